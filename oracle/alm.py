"""Explicit-flow (full-flow) augmented-Lagrangian max-flow solvers -- ORACLE (test infrastructure).

An INDEPENDENT way to reach the saddle point that the pseudo-flow iteration
converges to: every flow (source p_S, sink/intermediate p_v, spatial q_v) is
explicit, exactly the "full-flow" representation the paper reduces.
Derived by block-coordinate ascent on the augmented Lagrangian of the
primal-dual models, with u as the multipliers:

  Potts  (Eq. 3):   L_c = p_S + sum_L u_L r_L - c/2 sum_L r_L^2,
                             r_L = div q_L - p_S + p_L,  p_L <= D_L, |q_L| <= S_L.
  DAGMF  (Eq. 11): L_c = p_S + sum_v u_v r_v - c/2 sum_v r_v^2,
                             r_v = div q_v + p_v - sum_{P in v.P} w_(P,v) p_P,
                             p_L <= D_L for end labels only.

Shares nothing with pf_oracle.c (or the CUDA path); uses the oracle's numpy
grad/div from energy.py.
"""
from __future__ import annotations

import numpy as np

from .energy import _leaves, _order, div, grad


def _proj(q, S, cap):
    if cap == "l2":
        nrm = np.sqrt(np.sum(q * q, axis=0))
        f = np.where(nrm > S, S / np.where(nrm > 0, nrm, 1.0), 1.0)
        return q * f
    return np.clip(q, -S, S)


def potts_alm(D, S, ndim, iters, ca=0.3, ta=0.11, cap="l2"):
    """ALM for Eq. 3.  D: [K][...]; S: [K][...] per label capacity.  Returns (u, q, p_S)."""
    D = np.asarray(D, np.float64)
    K = D.shape[0]
    u = np.full(D.shape, 1.0 / K)
    q = np.zeros((K, ndim) + D.shape[1:])
    pS = np.min(D, axis=0)
    p = np.repeat(pS[None], K, axis=0).copy()
    for _ in range(iters):
        for L in range(K):
            dq = div(q[L], ndim)
            q[L] = _proj(q[L] + ta * grad(dq - pS + p[L] - u[L] / ca, ndim), S[L], cap)
            dq = div(q[L], ndim)
            p[L] = np.minimum(D[L], pS - dq + u[L] / ca)
        dqs = np.stack([div(q[L], ndim) for L in range(K)])
        pS = np.sum(p + dqs - u / ca, axis=0) / K + 1.0 / (K * ca)
        u = u - ca * (dqs - pS[None] + p)
    return u, q, pS


def dag_alm(D, S, num_nodes, parent, child, weight, ndim, iters, ca=0.3, ta=0.05, cap="l2"):
    """ALM for Eq. 11.  D: [NL][...]; S: [num_nodes][...] (row 0 unused).  Returns (u_leaves, q, p)."""
    D = np.asarray(D, np.float64)
    parent = [int(v) for v in parent]
    child = [int(v) for v in child]
    weight = [float(v) for v in weight]
    leaves = _leaves(num_nodes, parent)
    order = _order(num_nodes, parent, child)
    shape = D.shape[1:]
    kids = {v: [(c, w) for p, c, w in zip(parent, child, weight) if p == v] for v in range(num_nodes)}
    pars = {v: [(p, w) for p, c, w in zip(parent, child, weight) if c == v] for v in range(num_nodes)}
    # multipliers u_v for all non-source nodes, consistent start (u_L = 1/|L|)
    u = np.zeros((num_nodes,) + shape)
    for v in leaves:
        u[v] = 1.0 / len(leaves)
    for v in reversed(order):
        if v != 0 and v not in leaves:
            u[v] = sum(w * u[c] for c, w in kids[v])
    q = np.zeros((num_nodes, ndim) + shape)
    p = np.zeros((num_nodes,) + shape)
    p[0] = np.min(D, axis=0)
    dq = np.zeros((num_nodes,) + shape)

    def r(v):
        return dq[v] + p[v] - sum(w * p[P] for P, w in pars[v])

    for _ in range(iters):
        for v in order[1:]:
            q[v] = _proj(q[v] + ta * grad(r(v) - u[v] / ca, ndim), S[v], cap)
            dq[v] = div(q[v], ndim)
        for v in order:
            if v == 0:
                sw2 = sum(w * w for _, w in kids[0])
                num = (1.0 - sum(w * u[c] for c, w in kids[0])) / ca + sum(w * (r(c) + w * p[0]) for c, w in kids[0])
                p[0] = num / sw2
            elif v in leaves:
                p[v] = np.minimum(D[leaves.index(v)], u[v] / ca - dq[v] + sum(w * p[P] for P, w in pars[v]))
            else:
                sw2 = sum(w * w for _, w in kids[v])
                num = ((u[v] - sum(w * u[c] for c, w in kids[v])) / ca
                       - (dq[v] - sum(w * p[P] for P, w in pars[v]))
                       + sum(w * (r(c) + w * p[v]) for c, w in kids[v]))
                p[v] = num / (1.0 + sw2)
        res = {v: r(v) for v in order[1:]}
        for v in order[1:]:
            u[v] = u[v] - ca * res[v]
    return u[leaves], q[1:], p
