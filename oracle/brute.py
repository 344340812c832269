"""Exhaustive search over discrete labelings -- ORACLE (test infrastructure only).

Scores every one-hot labeling b: x -> L with the same discretized energy as
energy.primal (Eq. 1 P:53-59 / Eq. 9, intermediate labels
u_v = sum_B W_(v,B) u_B, W as defined at P:199-209), and returns the minimum.
"""
from __future__ import annotations

import itertools

import numpy as np

from .energy import _leaves, _order


def path_weights(num_nodes, parent, child, weight) -> np.ndarray:
    """W_(A,B) for all A and end labels B by the recursion of P:199-209."""
    leaves = _leaves(num_nodes, parent)
    order = _order(num_nodes, parent, child)
    W = np.zeros((num_nodes, len(leaves)))
    for v in reversed(order):
        if v in leaves:
            W[v, leaves.index(v)] = 1.0
        else:
            for p, c, w in zip(parent, child, weight):
                if int(p) == v:
                    W[v] += float(w) * W[int(c)]
    return W


def brute_force(D, S, num_nodes, parent, child, weight, ndim, cap="linf", max_states=2_000_000):
    """Return (E_min, labeling) over all |L|^V labelings.  D: [NL][nz][ny][nx]; S: [num_nodes][...]."""
    D = np.asarray(D, np.float64)
    NL = D.shape[0]
    shape = D.shape[1:]
    V = int(np.prod(shape))
    n = NL ** V
    if n > max_states:
        raise ValueError("instance too large for brute force")
    W = path_weights(num_nodes, parent, child, weight)  # [nodes][NL]
    B = np.array(list(itertools.product(range(NL), repeat=V)), dtype=np.int64)  # [n][V], x fastest flattening
    Dflat = D.reshape(NL, V)
    E = Dflat[B, np.arange(V)[None, :]].sum(axis=1)
    U = W[:, B]                                   # [nodes][n][V]: u_v(x) = W_(v, b(x))
    U = U.reshape((num_nodes, n) + shape)
    axes = {0: 3, 1: 2, 2: 1}                     # k -> axis of [node][n][z][y][x]
    for v in range(1, num_nodes):
        Sv = np.asarray(S[v], np.float64)
        acc = np.zeros((n,) + shape)
        for k in range(ndim):
            ax = axes[k]
            g = np.zeros((n,) + shape)
            lo = [slice(None)] * 4
            hi = [slice(None)] * 4
            lo[ax] = slice(0, shape[ax - 1] - 1)
            hi[ax] = slice(1, shape[ax - 1])
            g[tuple(lo)] = U[v][tuple(hi)] - U[v][tuple(lo)]
            acc += np.abs(g) if cap == "linf" else g * g
        nrm = acc if cap == "linf" else np.sqrt(acc)
        E += (nrm * Sv[None]).reshape(n, V).sum(axis=1)
    i = int(np.argmin(E))
    return float(E[i]), B[i].reshape(shape)
