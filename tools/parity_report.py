"""GPU-vs-oracle parity numbers (the values the -m gpu tests assert on), as JSON lines.

usage: python tools/parity_report.py   (needs a GPU; runs the oracle on the host)
* full-iteration parity on the scaled configs (C1 at full size);
* sampled parity at full size after a few iterations (window method, tests/helpers.py).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import phantoms as P  # noqa: E402
from helpers import bf16_rounded, solver_from_inputs, window_oracle  # noqa: E402


def full_case(name, dims, n, shift):
    cfg = P.config(name) if dims is None else P.config(name).resized(*dims)
    inp = P.generate(cfg)
    s = solver_from_inputs(inp, shift=shift)
    s.iterate(n)
    u, am = s.labeling()
    q = s.flows()
    info = s.kernel_info()
    s.close()
    t = time.perf_counter()
    ur, qr = O.run_inputs(inp, n, shift=shift)
    dt = time.perf_counter() - t
    return {"case": f"{name} {cfg.nx}x{cfg.ny}x{cfg.nz}", "iterations": n, "shift": ["min", "none"][shift],
            "max_abs_du": float(np.max(np.abs(u - ur))), "max_abs_dq": float(np.max(np.abs(q - qr))),
            "argmax_agree": float(np.mean(am == O.argmax(ur))), "voxels": int(cfg.V),
            "kernel_staged": info["staged"], "oracle_s": round(dt, 2)}


def bf16_case(name, dims, n):
    inp = bf16_rounded(P.generate(P.config(name).resized(*dims)))
    s = solver_from_inputs(inp, d_bf16=True)
    s.iterate(n)
    u, am = s.labeling()
    q = s.flows()
    s.close()
    ur, qr = O.run_inputs(inp, n)
    return {"case": f"{name} {dims[0]}x{dims[1]}x{dims[2]} D stored as bf16 (oracle on bf16-rounded D)",
            "iterations": n, "max_abs_du": float(np.max(np.abs(u - ur))), "max_abs_dq": float(np.max(np.abs(q - qr))),
            "argmax_agree": float(np.mean(am == O.argmax(ur)))}


def alm_case(name, dims, n):
    import paper_1501_07844_b200 as pf
    from oracle import alm as A
    inp = P.generate(P.config(name).resized(*dims))
    s = solver_from_inputs(inp, method=pf.PF_METHOD_EXPLICIT_ALM, c=0.3, tau=0.11)
    s.iterate(n)
    u, am = s.labeling()
    q = s.flows()
    s.close()
    K = inp.D.shape[0]
    S = (np.repeat(inp.s_field[None].astype(np.float64), K, axis=0) if inp.s_kind == "shared_field" else
         np.stack([np.full(inp.shape, float(inp.s_scalars[1 + l])) for l in range(K)]))
    ur, qr, _ = A.potts_alm(inp.D, S, inp.cfg.ndim, n, ca=0.3, ta=0.11)
    return {"case": f"{name} {dims[0]}x{dims[1]}x{dims[2]} explicit-flow ALM vs oracle/alm.py", "iterations": n,
            "max_abs_du": float(np.max(np.abs(u - ur))), "max_abs_dq": float(np.max(np.abs(q - qr))),
            "argmax_agree": float(np.mean(am == np.argmax(ur, axis=0)))}


def sampled_case(name, n=6):
    cfg = P.config(name) if name != "C5slab" else P.config("C5").resized(768, 768, 96, name="C5slab")
    inp = P.generate(cfg)
    s = solver_from_inputs(inp)
    s.iterate(n)
    u, _ = s.labeling()
    q = s.flows()
    zc = s.kernel_info()["z_chunk"]
    s.close()
    pts = [(0, 0, 0), (cfg.nx - 1, cfg.ny - 1, cfg.nz - 1), (31, 7, zc - 1), (32, 8, zc), (cfg.nx // 2, cfg.ny // 2,
                                                                                          cfg.nz // 2)]
    du = dq = 0.0
    agree = 0
    tot = 0
    for pt in pts:
        reg, ur, qr = window_oracle(cfg, pt, n, r=2)
        sl = tuple(slice(a, b) for a, b in reg)
        ug = u[(slice(None),) + sl].astype(np.float64)
        qg = q[(slice(None), slice(None)) + sl].astype(np.float64)
        du = max(du, float(np.max(np.abs(ug - ur))))
        dq = max(dq, float(np.max(np.abs(qg - qr))))
        agree += int(np.sum(np.argmax(ug, 0) == np.argmax(ur, 0)))
        tot += ur[0].size
    return {"case": f"{cfg.name} full size {cfg.nx}x{cfg.ny}x{cfg.nz} (sampled windows)", "iterations": n,
            "max_abs_du": du, "max_abs_dq": dq, "argmax_agree": agree / tot, "sampled_voxels": tot}


if __name__ == "__main__":
    cases = [("C1", None, 200, 0), ("C1", None, 200, 1), ("C2", (64, 64, 64), 300, 0), ("C2", (67, 45, 37), 300, 1),
             ("C3", (48, 40, 36), 300, 0), ("C4", (40, 40, 40), 300, 0), ("C4", (35, 70, 21), 80, 1),
             ("C5", (40, 36, 24), 200, 0), ("I2", (48, 40, 36), 300, 0), ("I2", (37, 29, 19), 300, 1)]
    for c in cases:
        print(json.dumps(full_case(*c)), flush=True)
    for c in [("C2", (67, 45, 37), 300), ("C5", (40, 36, 24), 200)]:
        print(json.dumps(bf16_case(*c)), flush=True)
    for c in [("C1", (64, 64, 1), 200), ("C2", (37, 29, 21), 100)]:
        print(json.dumps(alm_case(*c)), flush=True)
    for name in ("C2", "C3", "C4", "C5slab", "I2"):
        print(json.dumps(sampled_case(name)), flush=True)
