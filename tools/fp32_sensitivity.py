"""Diagnostic (not part of the oracle): an independent numpy float32 re-implementation of Alg. 2, compared with
the fp64 oracle, showing that the literal listing (SHIFT_NONE) on the C4-shaped DAG separates fp32 from fp64
trajectories after ~60-100 iterations (max|dq| 1e-7 at 50, 8e-5 at 100, 8e-4 at 150) -- the same pattern as the
GPU kernel, so it is the conditioning of that reading, not a kernel defect.  usage: PYTHONPATH=. python tools/fp32_sensitivity.py"""
import numpy as np, phantoms as P, oracle as O
from oracle import energy as Eo
def grad(f):  # f [z][y][x]
    g = np.zeros((3,)+f.shape, f.dtype)
    g[0][:,:,:-1] = f[:,:,1:]-f[:,:,:-1]; g[1][:,:-1,:] = f[:,1:,:]-f[:,:-1,:]; g[2][:-1] = f[1:]-f[:-1]
    return g
def div(q):
    out = q[0] + q[1] + q[2]
    out = q[0].copy(); out[:,:,1:] -= q[0][:,:,:-1]
    t = q[1].copy(); t[:,1:,:] -= q[1][:,:-1,:]
    t2 = q[2].copy(); t2[1:] -= q[2][:-1]
    return (out + t) + t2
def run(inp, n, dt, shift):
    g = inp.graph; leaves = g.leaves(); NL=len(leaves)
    order = O.topo_order(g.num_nodes, g.parent, g.child, g.weight)
    D = inp.D.astype(dt); S = [None]+[f.astype(dt) for f in inp.s_fields()[1:]]
    u = np.full((NL,)+inp.shape, 1.0/NL, dt); q = np.zeros((g.num_nodes-1,3)+inp.shape, dt)
    c = dt(0.25); ctau = dt(0.025)
    for it in range(n):
        d = [None]*g.num_nodes
        for v in range(1,g.num_nodes): d[v] = div(q[v-1])
        for s_, v in enumerate(leaves): d[v] = D[s_] + d[v]
        for L in order[1:]:
            for p_, c_, w in zip(g.parent, g.child, g.weight):
                if p_ == L: d[c_] = d[c_] + dt(w)*d[L]
        m = np.min([d[v] for v in leaves], axis=0) if shift == 0 else dt(0)
        ut = np.stack([u[s_]*np.exp(-(d[v]-m)/c) for s_, v in enumerate(leaves)])
        a = ut.sum(0); u = ut/a; u[u < np.finfo(np.float32).tiny] = 0
        M = [None]*g.num_nodes
        for s_, v in enumerate(leaves): M[v] = ut[s_]
        for v in range(1, g.num_nodes):
            if v not in leaves: M[v] = np.zeros(inp.shape, dt)
        for L in reversed(order[1:]):
            for p_, c_, w in zip(g.parent, g.child, g.weight):
                if c_ == L and p_ != 0: M[p_] = M[p_] + dt(w)*M[L]
        for v in range(1, g.num_nodes):
            h = q[v-1] - ctau*grad(M[v])
            nrm = np.sqrt((h.astype(np.float64)**2).sum(0)).astype(dt)
            f = np.where(nrm > S[v], S[v]/np.where(nrm > 0, nrm, 1), 1).astype(dt)
            q[v-1] = h*f
    return u, q
inp = P.generate(P.config("C4").resized(35,70,21))
for n in (50, 100, 150):
    u32, q32 = run(inp, n, np.float32, 1)
    ur, qr = O.run_inputs(inp, n, shift=1)
    dq = np.abs(q32 - qr); i = np.unravel_index(np.argmax(dq), dq.shape)
    print(n, "f32-numpy vs oracle du", np.abs(u32-ur).max(), "dq", dq.max(), "at", i)
