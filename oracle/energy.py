"""Primal and dual energies of the discretized models -- ORACLE (test infrastructure only).

Discretization (reading R4): nabla = forward differences with 0 at the last index,
div = -nabla^T (backward differences with q(-1) = 0).  Norms (reading R5):
capacity l2 <-> isotropic TV |nabla u|_2; capacity l-inf box <-> anisotropic TV
|nabla u|_1.

Arrays use the boundary layout: u [NL][nz][ny][nx], q [node-1][ndim][nz][ny][nx],
S per node [num_nodes][nz][ny][nx] (row 0 unused), fp64.
"""
from __future__ import annotations

from typing import List

import numpy as np

_AX = {0: 2, 1: 1, 2: 0}   # component k (x, y, z) -> numpy axis of a [z][y][x] volume


def grad(f: np.ndarray, ndim: int) -> np.ndarray:
    """(nabla f)^k(x) = f(x+e_k) - f(x), 0 at the last index (reading R4)."""
    g = np.zeros((ndim,) + f.shape, dtype=np.float64)
    for k in range(ndim):
        ax = _AX[k]
        sl_lo = [slice(None)] * 3
        sl_hi = [slice(None)] * 3
        sl_lo[ax] = slice(0, f.shape[ax] - 1)
        sl_hi[ax] = slice(1, f.shape[ax])
        g[k][tuple(sl_lo)] = f[tuple(sl_hi)] - f[tuple(sl_lo)]
    return g


def div(q: np.ndarray, ndim: int) -> np.ndarray:
    """div q = sum_k q^k(x) - q^k(x-e_k), q^k(-1) = 0 (reading R4)."""
    out = np.zeros(q.shape[1:], dtype=np.float64)
    for k in range(ndim):
        ax = _AX[k]
        out += q[k]
        sl_lo = [slice(None)] * 3
        sl_hi = [slice(None)] * 3
        sl_lo[ax] = slice(0, q.shape[1 + ax] - 1)
        sl_hi[ax] = slice(1, q.shape[1 + ax])
        out[tuple(sl_hi)] -= q[k][tuple(sl_lo)]
    return out


def _leaves(num_nodes: int, parent) -> List[int]:
    has_child = set(int(p) for p in parent)
    return [v for v in range(1, num_nodes) if v not in has_child]


def _order(num_nodes, parent, child):
    """Topological order (Kahn, lowest id first) -- own copy, numpy side."""
    indeg = [0] * num_nodes
    for c in child:
        indeg[int(c)] += 1
    placed, order = [False] * num_nodes, []
    for _ in range(num_nodes):
        v = next(v for v in range(num_nodes) if not placed[v] and indeg[v] == 0)
        placed[v] = True
        order.append(v)
        for p, c in zip(parent, child):
            if int(p) == v:
                indeg[int(c)] -= 1
    return order


def all_labels(u: np.ndarray, num_nodes: int, parent, child, weight) -> np.ndarray:
    """u_v for every node: end labels given, u_v = sum_{c in v.C} w u_c (Eq. 9), bottom-up."""
    leaves = _leaves(num_nodes, parent)
    out = np.zeros((num_nodes,) + u.shape[1:], dtype=np.float64)
    for slot, v in enumerate(leaves):
        out[v] = u[slot]
    for v in reversed(_order(num_nodes, parent, child)):
        if v in leaves:
            continue
        acc = np.zeros(u.shape[1:], dtype=np.float64)
        for p, c, w in zip(parent, child, weight):
            if int(p) == v:
                acc += float(w) * out[int(c)]
        out[v] = acc
    return out


def primal(u, D, S, num_nodes, parent, child, weight, ndim, cap="l2") -> float:
    """E(u) = sum_{L in L} <D_L, u_L> + sum_{v != S} <S_v, |nabla u_v|>  (Eq. 1; Eq. 9)."""
    U = all_labels(u, num_nodes, parent, child, weight)
    E = float(np.sum(D.astype(np.float64) * u))
    for v in range(1, num_nodes):
        g = grad(U[v], ndim)
        nrm = np.sqrt(np.sum(g * g, axis=0)) if cap == "l2" else np.sum(np.abs(g), axis=0)
        E += float(np.sum(S[v] * nrm))
    return E


def excess(q, D, num_nodes, parent, child, weight, ndim) -> np.ndarray:
    """d_L for every node: d_S = 0; d_L = [D_L] + div q_L + sum_{L' in L.P} w d_L'."""
    leaves = _leaves(num_nodes, parent)
    d = np.zeros((num_nodes,) + D.shape[1:], dtype=np.float64)
    order = _order(num_nodes, parent, child)
    for v in order[1:]:
        acc = div(q[v - 1], ndim)
        if v in leaves:
            acc = acc + D[leaves.index(v)]
        for p, c, w in zip(parent, child, weight):
            if int(c) == v and int(p) != 0:
                acc = acc + float(w) * d[int(p)]
        d[v] = acc
    return d


def dual(q, D, num_nodes, parent, child, weight, ndim) -> float:
    """F(q) = integral of min_{L in L} d_L(x)  (Eq. 4; Eq. 13)."""
    d = excess(q, D, num_nodes, parent, child, weight, ndim)
    leaves = _leaves(num_nodes, parent)
    return float(np.sum(np.min(d[leaves], axis=0)))


def potts_graph_arrays(K: int):
    return K + 1, np.zeros(K, np.int32), np.arange(1, K + 1, dtype=np.int32), np.ones(K)
