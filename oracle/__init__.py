"""CPU ORACLE for arXiv 1501.07844 (pseudo-flow continuous max-flow) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_1501_07844_b200``) never imports it; the two share no code.

Contents
  * ``potts_iterate`` / ``dag_iterate``: Algorithms 1 and 2 (PAPER.md P:144-153,
    P:279-305), plain C in fp64 (``pf_oracle.c``), one whole-field pass per
    listing line.
  * ``energy``: primal E(u) (Eq. 1, Eq. 9) and pseudo-flow dual
    F(q) (Eq. 4, Eq. 13), numpy fp64.
  * ``alm``: independent explicit-flow augmented-Lagrangian max-flow solvers
    derived from the primal-dual models Eq. 3 and Eq. 11.
  * ``brute``: exhaustive search over discrete labelings.

Parity pins for every function are in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

SHIFT_MIN, SHIFT_NONE = 0, 1
U_FLOOR = 0.0          # reading R18: no floor (paper-exact); u_floor > 0 is an opt-in diagnostic only
FP32_NORMAL_MIN = 2.0 ** -126
CAP_L2, CAP_LINF = 0, 1


def build(force: bool = False) -> str:
    """Compile pf_oracle.c with plain IEEE semantics (no fast-math, no contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC",
                               "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64, i32, dp, ip = ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int)
        lib.oracle_potts.restype = i64
        lib.oracle_potts.argtypes = [i32, i64, i64, i64, i32, dp, dp, dp, dp, ctypes.c_double, ctypes.c_double,
                                     i32, i32, i32, ctypes.c_double]
        lib.oracle_dag.restype = i64
        lib.oracle_dag.argtypes = [i32, i64, i64, i64, i32, i32, ip, ip, dp, dp, dp, dp, dp, ctypes.c_double,
                                   ctypes.c_double, i32, i32, i32, ctypes.c_double]
        lib.oracle_ishikawa.restype = i64
        lib.oracle_ishikawa.argtypes = [i32, i64, i64, i64, i32, dp, dp, dp, dp, ctypes.c_double, ctypes.c_double,
                                        i32, i32, i32, ctypes.c_double]
        lib.oracle_topo_order.restype = i32
        lib.oracle_topo_order.argtypes = [i32, i32, ip, ip, dp, ip]
        lib.oracle_grad.restype = i32
        lib.oracle_grad.argtypes = [i32, i64, i64, i64, dp, i32, dp]
        lib.oracle_div.restype = i32
        lib.oracle_div.argtypes = [i32, i64, i64, i64, dp, dp]
        lib.oracle_set_threads.restype = None
        lib.oracle_set_threads.argtypes = [i32]
        lib.oracle_project.restype = i32
        lib.oracle_project.argtypes = [i32, i64, i64, i64, dp, dp, i32]
        _lib = lib
    return _lib


def set_threads(n: int) -> None:
    """Threads for the oracle's whole-field passes (default 1, the plain single-threaded oracle).  Every pass
    is a per-voxel pure function, so the results are bit-identical for any n (tests/test_oracle_pins.py)."""
    _load().oracle_set_threads(int(n))


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


class OracleError(RuntimeError):
    pass


def _status(st: int):
    if st == 0:
        return
    if st == -1000000000000:
        raise OracleError("invalid arguments")
    raise OracleError(f"numerical collapse a(x) <= 0 at voxel {-1 - st}")


def init_state(num_leaves: int, num_flow_nodes: int, shape: Sequence[int], ndim: int):
    """u_L = 1/|L|; q = 0 (reading R8).  shape = (nz, ny, nx)."""
    u = np.full((num_leaves,) + tuple(shape), 1.0 / num_leaves, dtype=np.float64)
    q = np.zeros((num_flow_nodes, ndim) + tuple(shape), dtype=np.float64)
    return u, q


def potts_iterate(D: np.ndarray, S: np.ndarray, u: np.ndarray, q: np.ndarray, ndim: int, c: float, tau: float,
                  niter: int, shift: int = SHIFT_MIN, cap: int = CAP_L2, u_floor: float = U_FLOOR):
    """Algorithm 1 in place.  D,S,u: [K][nz][ny][nx]; q: [K][ndim][nz][ny][nx] (fp64, C order)."""
    K, nz, ny, nx = D.shape
    st = _load().oracle_potts(ndim, nx, ny, nz, K, _dp(D), _dp(S), _dp(u), _dp(q), c, tau, shift, cap, niter,
                              u_floor)
    _status(st)
    return u, q


def dag_iterate(num_nodes: int, parent, child, weight, D: np.ndarray, S: np.ndarray, u: np.ndarray, q: np.ndarray,
                ndim: int, c: float, tau: float, niter: int, shift: int = SHIFT_MIN, cap: int = CAP_L2,
                u_floor: float = U_FLOOR):
    """Algorithm 2 in place.  D,u: [NL][...]; S: [num_nodes][...] (row 0 unused); q: [num_nodes-1][ndim][...]."""
    NL, nz, ny, nx = D.shape
    par = np.ascontiguousarray(parent, dtype=np.int32)
    chi = np.ascontiguousarray(child, dtype=np.int32)
    w = np.ascontiguousarray(weight, dtype=np.float64)
    st = _load().oracle_dag(ndim, nx, ny, nz, num_nodes, len(par), _ip(par), _ip(chi), _dp(w), _dp(D), _dp(S),
                            _dp(u), _dp(q), c, tau, shift, cap, niter, u_floor)
    _status(st)
    return u, q


def ishikawa_iterate(D: np.ndarray, S: np.ndarray, u: np.ndarray, q: np.ndarray, ndim: int, c: float, tau: float,
                     niter: int, shift: int = SHIFT_MIN, cap: int = CAP_L2, u_floor: float = U_FLOOR):
    """Algorithm 3 in place.  D,u: [N+1][...]; S: [N][...] (level flows 1..N); q: [N][ndim][...]."""
    NL, nz, ny, nx = D.shape
    st = _load().oracle_ishikawa(ndim, nx, ny, nz, NL - 1, _dp(D), _dp(S), _dp(u), _dp(q), c, tau, shift, cap,
                                 niter, u_floor)
    _status(st)
    return u, q


def topo_order(num_nodes: int, parent, child, weight) -> Optional[List[int]]:
    """O by Kahn's algorithm with lowest-id tie-break; None if invalid."""
    par = np.ascontiguousarray(parent, dtype=np.int32)
    chi = np.ascontiguousarray(child, dtype=np.int32)
    w = np.ascontiguousarray(weight, dtype=np.float64)
    out = np.zeros(num_nodes, dtype=np.int32)
    ok = _load().oracle_topo_order(num_nodes, len(par), _ip(par), _ip(chi), _dp(w), _ip(out))
    return [int(v) for v in out] if ok else None


def grad(f: np.ndarray, k: int, ndim: int) -> np.ndarray:
    """(nabla f)^k of a [nz][ny][nx] fp64 volume (C operator; reading R4)."""
    f = np.ascontiguousarray(f, dtype=np.float64)
    g = np.empty_like(f)
    nz, ny, nx = f.shape
    assert _load().oracle_grad(ndim, nx, ny, nz, _dp(f), k, _dp(g))
    return g


def div(q: np.ndarray, ndim: int) -> np.ndarray:
    """div q of a [ndim][nz][ny][nx] fp64 flow (C operator; reading R4)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    out = np.empty(q.shape[1:], dtype=np.float64)
    nz, ny, nx = q.shape[1:]
    assert _load().oracle_div(ndim, nx, ny, nz, _dp(q), _dp(out))
    return out


def project(q: np.ndarray, S: np.ndarray, ndim: int, cap: int = CAP_L2) -> np.ndarray:
    """Proj_{|q(x)| <= S(x)} of a [ndim][nz][ny][nx] flow (C operator; readings R5, R14)."""
    q = np.array(q, dtype=np.float64, order="C")
    S = np.ascontiguousarray(S, dtype=np.float64)
    nz, ny, nx = q.shape[1:]
    assert _load().oracle_project(ndim, nx, ny, nz, _dp(q), _dp(S), cap)
    return q


def argmax(u: np.ndarray) -> np.ndarray:
    """Thresholded labeling: per-voxel argmax over end labels, ties -> lowest index."""
    return np.argmax(u, axis=0).astype(np.uint8)


def run_inputs(inp, niter: int, shift: int = SHIFT_MIN, cap: Optional[int] = None, c: Optional[float] = None,
               tau: Optional[float] = None, state=None, u_floor: float = U_FLOOR):
    """Run the oracle on a phantoms.Inputs object from the initial state (or `state`)."""
    cfg, g = inp.cfg, inp.graph
    cap = (CAP_L2 if cfg.cap == "l2" else CAP_LINF) if cap is None else cap
    c = cfg.c if c is None else c
    tau = cfg.tau if tau is None else tau
    D = np.ascontiguousarray(inp.D, dtype=np.float64)
    fields = inp.s_fields()
    S = np.zeros((g.num_nodes,) + inp.shape, dtype=np.float64)
    for v in range(1, g.num_nodes):
        S[v] = fields[v]
    NL = D.shape[0]
    if state is None:
        u, q = init_state(NL, g.num_nodes - 1, inp.shape, cfg.ndim)
    else:
        u, q = state
    if cfg.kind == "potts":
        potts_iterate(D, np.ascontiguousarray(S[1:]), u, q, cfg.ndim, c, tau, niter, shift, cap, u_floor)
    elif cfg.kind == "ishikawa":
        # Alg. 3 on the level flows (node ids 1..N); end labels (ids N+1..) carry no flow and stay 0
        N = NL - 1
        ishikawa_iterate(D, np.ascontiguousarray(S[1:N + 1]), u, q[:N], cfg.ndim, c, tau, niter, shift, cap, u_floor)
    else:
        dag_iterate(g.num_nodes, g.parent, g.child, g.weight.astype(np.float64), D, S, u, q, cfg.ndim, c, tau,
                    niter, shift, cap, u_floor)
    return u, q
