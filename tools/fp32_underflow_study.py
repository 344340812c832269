"""Diagnostic (not part of the oracle, not on the product path): how far an fp32 execution of Alg. 2 can
follow the paper-exact fp64 oracle (u_floor = 0) on the HMF (C3) shapes where labels die and revive.

Three fp32 storage/arithmetic variants of the label update (P:290-293 / Eq. 15), everything else fp32:
  flush  -- normalised u < FLT_MIN set to 0 and exp results flushed (round-1 kernel: ex2.approx.ftz + floor)
  subn   -- IEEE fp32 with subnormals kept (no FTZ anywhere)
  log2T16 -- log2T with the stored lambda rounded to binary16 (pf_config.u_half)
  log2   -- u stored as lambda = log2 u in fp32; u~ = 2^(lambda + (m - d) log2(e)/c) for the sums/masses,
            lambda' = lambda + (m - d) log2(e)/c - log2(a)  (no underflow of the stored state)
usage: PYTHONPATH=. python tools/fp32_underflow_study.py [C3 33 17 9 300 0] ...
"""
import sys

import numpy as np

import oracle as O
import phantoms as P

f32 = np.float32
TINY = np.finfo(np.float32).tiny
import os
MODES = os.environ.get("MODES", "flush,subn,log2,log2T").split(",")


def grad(f):
    g = np.zeros((3,) + f.shape, f.dtype)
    g[0][:, :, :-1] = f[:, :, 1:] - f[:, :, :-1]
    g[1][:, :-1, :] = f[:, 1:, :] - f[:, :-1, :]
    g[2][:-1] = f[1:] - f[:-1]
    return g


def div(q):
    a = q[0].copy(); a[:, :, 1:] -= q[0][:, :, :-1]
    b = q[1].copy(); b[:, 1:, :] -= q[1][:, :-1, :]
    c = q[2].copy(); c[1:] -= q[2][:-1]
    return (a + b) + c


def exp2_f32(x, flush):
    y = np.exp2(x.astype(np.float64)).astype(f32)   # correctly rounded-ish, subnormals kept
    if flush:
        y[y < TINY] = 0
    return y


def run32(inp, n, shift, mode):
    g = inp.graph
    leaves = g.leaves()
    NL = len(leaves)
    order = O.topo_order(g.num_nodes, g.parent, g.child, g.weight)
    D = inp.D.astype(f32)
    S = [None] + [f.astype(f32) for f in inp.s_fields()[1:]]
    if mode.startswith("log2"):
        lam = np.full((NL,) + inp.shape, np.log2(1.0 / NL), f32)
    else:
        u = np.full((NL,) + inp.shape, 1.0 / NL, f32)
    q = np.zeros((g.num_nodes - 1, 3) + inp.shape, f32)
    k2 = f32(1.4426950408889634 / inp.cfg.c)
    ctau = f32(inp.cfg.c * inp.cfg.tau)
    with np.errstate(divide="ignore", over="ignore", under="ignore", invalid="ignore"):
        for _ in range(n):
            d = [None] * g.num_nodes
            for v in range(1, g.num_nodes):
                d[v] = div(q[v - 1])
            for s_, v in enumerate(leaves):
                d[v] = D[s_] + d[v]
            for L in order[1:]:
                for p_, c_, w in zip(g.parent, g.child, g.weight):
                    if p_ == L:
                        d[c_] = d[c_] + f32(w) * d[L]
            m = np.min([d[v] for v in leaves], axis=0) if shift == 0 else f32(0)
            if mode == "log2":
                t = np.stack([lam[s_] + (m - d[v]) * k2 for s_, v in enumerate(leaves)]).astype(f32)
                ut = exp2_f32(t, False)
                a = ut.sum(0, dtype=f32)
                lam = (t - np.log2(a.astype(np.float64)).astype(f32)).astype(f32)
            elif mode in ("log2T", "log2T16"):   # the kernel's form: max shift T, e = 2^(t-T) in (0,1], s = sum e in [1,K]
                t = np.stack([lam[s_] + (m - d[v]) * k2 for s_, v in enumerate(leaves)]).astype(f32)
                T = t.max(0)
                r = (t - T).astype(f32)
                e = exp2_f32(r, True)
                s = e.sum(0, dtype=f32)
                lam = (r - np.log2(s.astype(np.float64)).astype(f32)).astype(f32)
                if mode == "log2T16":   # pf_config.u_half: the stored lambda rounded to binary16
                    lam = lam.astype(np.float16).astype(f32)
                ut = (e * exp2_f32(T, True)).astype(f32)
            else:
                fl = mode == "flush"
                ut = np.stack([u[s_] * exp2_f32((m - d[v]) * k2, fl) for s_, v in enumerate(leaves)]).astype(f32)
                a = ut.sum(0, dtype=f32)
                u = (ut * (f32(1) / a)).astype(f32)
                if fl:
                    u[u < TINY] = 0
            M = [None] * g.num_nodes
            for s_, v in enumerate(leaves):
                M[v] = ut[s_]
            for v in range(1, g.num_nodes):
                if v not in leaves:
                    M[v] = np.zeros(inp.shape, f32)
            for L in reversed(order[1:]):
                for p_, c_, w in zip(g.parent, g.child, g.weight):
                    if c_ == L and p_ != 0:
                        M[p_] = M[p_] + f32(w) * M[L]
            for v in range(1, g.num_nodes):
                h = q[v - 1] - ctau * grad(M[v])
                nrm = np.sqrt((h.astype(np.float64) ** 2).sum(0)).astype(f32)
                fac = np.where(nrm > S[v], S[v] / np.where(nrm > 0, nrm, 1), 1).astype(f32)
                q[v - 1] = h * fac
    if mode.startswith("log2"):
        u = np.exp2(lam.astype(np.float64))
    return u, q


def main(argv):
    cases = [argv[i:i + 6] for i in range(0, len(argv), 6)] or [["C3", "33", "17", "9", "300", "0"]]
    for name, nx, ny, nz, n, shift in cases:
        nx, ny, nz, n, shift = int(nx), int(ny), int(nz), int(n), int(shift)
        inp = P.generate(P.config(name).resized(nx, ny, nz))
        ur, qr = O.run_inputs(inp, n, shift=shift, u_floor=0.0)
        print(f"{name} {nx}x{ny}x{nz} n={n} shift={'MIN' if shift == 0 else 'NONE'}  min u (fp64) = {ur.min():.3g}")
        for mode in MODES:
            u, q = run32(inp, n, shift, mode)
            du = np.abs(u - ur)
            dq = np.abs(q - qr)
            am = np.mean(np.argmax(u, 0) == np.argmax(ur, 0))
            print(f"  {mode:6s} max|du| {du.max():.3g}  max|dq| {dq.max():.3g}  voxels du>1e-4: "
                  f"{int((du.max(0) > 1e-4).sum())}/{du[0].size}  argmax {am * 100:.4f}%", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
