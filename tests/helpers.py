"""Shared test helpers: build a GPU solver from phantoms.Inputs and compare against the oracle."""
import numpy as np

import phantoms as P

CAP = {"l2": 0, "linf": 1}


def solver_from_inputs(inp, shift=0, cap=None, check_every=10, slab=None, c=None, tau=None, device_inputs=False,
                       d_bf16=False, method=0, u_half=False, tblock=0):
    import paper_1501_07844_b200 as pf

    cfg, g = inp.cfg, inp.graph
    nz = cfg.nz
    z0, z1 = (0, nz) if slab is None else slab
    zt = min(z1 + 1, nz)
    wz0 = inp.window[0]
    D = [np.ascontiguousarray(inp.D[l, z0 - wz0:zt - wz0]) for l in range(inp.D.shape[0])]
    kw = {}
    if cfg.kind == "ishikawa":   # level nodes carry the shared field, end labels no flow (factor 0)
        factors = np.zeros(g.num_nodes, np.float32)
        factors[1:len(D)] = 1.0
        kw["s_scaled"] = (factors, np.ascontiguousarray(inp.s_field[z0 - wz0:z1 - wz0]))
    elif inp.s_kind == "shared_field":
        kw["s_shared"] = np.ascontiguousarray(inp.s_field[z0 - wz0:z1 - wz0])
    elif inp.s_kind == "field_per_node":
        kw["s_fields"] = [np.ascontiguousarray(f[z0 - wz0:z1 - wz0]) for f in inp.s_fields()[1:]]
    else:
        kw["s_scalars"] = inp.s_scalars
    if device_inputs:
        import torch
        D = [torch.from_numpy(d).cuda() for d in D]
        for k in ("s_shared",):
            if k in kw:
                kw[k] = torch.from_numpy(kw[k]).cuda()
        if "s_scaled" in kw:
            kw["s_scaled"] = (kw["s_scaled"][0], torch.from_numpy(kw["s_scaled"][1]).cuda())
    cap = CAP[cfg.cap] if cap is None else cap
    return pf.Solver((cfg.nx, cfg.ny, cfg.nz), cfg.ndim, (g.num_nodes, g.parent, g.child, g.weight), D,
                     c=cfg.c if c is None else c, tau=cfg.tau if tau is None else tau, cap=cap, shift=shift,
                     check_every=check_every, slab=None if slab is None else (z0, z1), d_bf16=d_bf16, u_half=u_half, tblock=tblock,
                     method=method, **kw)


def bf16_rounded(inp):
    """`inp` with its data terms rounded to bf16 (round-to-nearest-even) -- the problem a solver created
    with d_bf16 solves (pf_config.d_bf16).  Input preprocessing only: the oracle then runs unchanged."""
    b = np.ascontiguousarray(inp.D, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    D = b.astype(np.uint32).view(np.float32)
    out = P.Inputs(inp.cfg, inp.graph, inp.window, D, inp.s_kind, inp.s_scalars, inp.s_field, inp.intensity)
    return out


def compare(u_gpu, q_gpu, u_ref, q_ref, tol=1e-4, argmax_frac=0.9999):
    du = float(np.max(np.abs(u_gpu.astype(np.float64) - u_ref))) if u_ref.size else 0.0
    dq = float(np.max(np.abs(q_gpu.astype(np.float64) - q_ref))) if q_ref.size else 0.0
    am = np.argmax(u_gpu, axis=0) == np.argmax(u_ref, axis=0)
    frac = float(np.mean(am))
    assert du <= tol and dq <= tol, f"max|du|={du:.3g} max|dq|={dq:.3g} (tol {tol})"
    assert frac >= argmax_frac, f"argmax agreement {frac}"
    return du, dq, frac


def with_field_per_node(inp, seed=5):
    """Variant of `inp` whose capacities are one random field per non-source node (PF_S_FIELD_PER_NODE)."""
    r = np.random.default_rng(seed)
    fields = [None] + [r.uniform(0.0, 0.2, size=inp.shape).astype(np.float32) for _ in range(inp.graph.num_nodes - 1)]
    out = P.Inputs(inp.cfg, inp.graph, inp.window, inp.D, "field_per_node", None, None, inp.intensity)
    out.s_fields = lambda: fields
    return out


def window_around(cfg, point, radius):
    """Window (z0, z1, y0, y1, x0, x1) of half-width `radius` around point (x, y, z), clipped to the volume."""
    x, y, z = point
    return (max(0, z - radius), min(cfg.nz, z + radius + 1), max(0, y - radius), min(cfg.ny, y + radius + 1),
            max(0, x - radius), min(cfg.nx, x + radius + 1))


def exact_region(cfg, window, point, n, r):
    """Sub-box of `window` (global coords) whose oracle values after n iterations do not depend on the
    window's artificial edges: at distance > n from every artificial edge, and within r of `point`."""
    z0, z1, y0, y1, x0, x1 = window
    out = []
    for (lo, hi, c, N) in ((z0, z1, point[2], cfg.nz), (y0, y1, point[1], cfg.ny), (x0, x1, point[0], cfg.nx)):
        a = lo if lo == 0 else lo + n + 1
        b = hi if hi == N else hi - n - 1
        out.append((max(a, c - r), min(b, c + r + 1)))
    return out


def window_oracle(cfg, point, n, r=2, shift=0):
    """Oracle u, q after n iterations on a window around `point` (inputs regenerated for the window).
    Returns (region as ((z0,z1),(y0,y1),(x0,x1)) global, u_ref, q_ref) restricted to the exact region."""
    import oracle as O
    win = window_around(cfg, point, n + 1 + r)
    inp = P.generate(cfg, win)
    u, q = O.run_inputs(inp, n, shift=shift)
    reg = exact_region(cfg, win, point, n, r)
    sl = tuple(slice(a - w0, b - w0) for (a, b), w0 in zip(reg, (win[0], win[2], win[4])))
    return reg, u[(slice(None),) + sl], q[(slice(None), slice(None)) + sl]
