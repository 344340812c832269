"""B200-native pseudo-flow continuous max-flow (arXiv 1501.07844) -- Python binding of libpf.so.

Argument marshalling only: every step of the hot path runs in the library's sm_100a
kernels (paper_1501_07844_b200/csrc).  The C-ABI is declared in include/pf.h; the
functions below carry the same names and semantics.  There is no CPU fallback: if
libpf.so is missing or cannot be loaded, importing this package raises.

Arrays may be numpy arrays (host) or CUDA torch tensors (device); they are passed as
raw pointers and copied by the library.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PF_LIB selects another in-tree build of the same library (A/B timing of kernel variants in one run;
# tools/ab.py).  The default is the library __graft_entry__.build() produces.
LIB_PATH = os.path.join(_HERE, os.environ.get("PF_LIB", "libpf.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

PF_OK, PF_ERR_INVALID, PF_ERR_GRAPH, PF_ERR_OOM, PF_ERR_CUDA, PF_ERR_UNSUPPORTED, PF_ERR_NUMERIC, PF_ERR_STATE = range(8)
PF_CAP_L2, PF_CAP_LINF = 0, 1
PF_METHOD_PSEUDO_FLOW, PF_METHOD_EXPLICIT_ALM = 0, 1
PF_SHIFT_MIN, PF_SHIFT_NONE = 0, 1
PF_S_SCALAR_PER_NODE, PF_S_SHARED_FIELD, PF_S_FIELD_PER_NODE, PF_S_SCALED_FIELD = 0, 1, 2, 3
_STATUS = {1: "PF_ERR_INVALID", 2: "PF_ERR_GRAPH", 3: "PF_ERR_OOM", 4: "PF_ERR_CUDA", 5: "PF_ERR_UNSUPPORTED",
           6: "PF_ERR_NUMERIC", 7: "PF_ERR_STATE"}

EXPORTED = ["pf_create", "pf_reset", "pf_set_step", "pf_iterate", "pf_run", "pf_iterate_phase", "pf_get_node_labeling",
            "pf_link_slabs", "pf_iterate_linked", "pf_ipc_export", "pf_ipc_link", "pf_ipc_step", "pf_get_labeling", "pf_get_flows", "pf_get_state", "pf_set_state", "pf_get_energy",
            "pf_iterations", "pf_set_stream", "pf_set_reserved_sms", "pf_halo_regions", "pf_exchange_local", "pf_get_kernel_info",
            "pf_destroy", "pf_last_error", "pf_version"]


class pf_dims(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64)]


class pf_graph(ctypes.Structure):
    _fields_ = [("num_nodes", ctypes.c_int32), ("num_edges", ctypes.c_int32),
                ("parent", ctypes.POINTER(ctypes.c_int32)), ("child", ctypes.POINTER(ctypes.c_int32)),
                ("weight", ctypes.POINTER(ctypes.c_float))]


class pf_smoothness(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("scalars", ctypes.POINTER(ctypes.c_float)),
                ("fields", ctypes.POINTER(ctypes.c_void_p))]


class pf_config(ctypes.Structure):
    _fields_ = [("c", ctypes.c_float), ("tau", ctypes.c_float), ("cap", ctypes.c_int32), ("shift", ctypes.c_int32),
                ("check_every", ctypes.c_int32), ("d_bf16", ctypes.c_int32), ("ipc", ctypes.c_int32),
                ("method", ctypes.c_int32), ("u_half", ctypes.c_int32), ("tblock", ctypes.c_int32)]


class pf_ipc_slab(ctypes.Structure):
    _fields_ = [("u", (ctypes.c_uint8 * 64) * 2), ("q", (ctypes.c_uint8 * 64) * 2), ("event", ctypes.c_uint8 * 64),
                ("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nzl", ctypes.c_int64), ("z0", ctypes.c_int64),
                ("pitch", ctypes.c_int64), ("NF", ctypes.c_int32), ("NL", ctypes.c_int32), ("tile_y", ctypes.c_int32),
                ("cluster", ctypes.c_int32), ("cur", ctypes.c_int32), ("inbox", ctypes.c_uint8 * 64),
                ("seq", ctypes.c_uint32), ("u_half", ctypes.c_int32)]


class pf_slab(ctypes.Structure):
    _fields_ = [("z_begin", ctypes.c_int64), ("z_end", ctypes.c_int64)]


class pf_halo(ctypes.Structure):
    _fields_ = [("send_down_u", ctypes.c_void_p), ("recv_up_u", ctypes.c_void_p),
                ("send_down_q", ctypes.c_void_p), ("recv_up_q", ctypes.c_void_p),
                ("send_up_qz", ctypes.c_void_p), ("recv_down_qz", ctypes.c_void_p),
                ("bytes_u", ctypes.c_int64), ("bytes_q", ctypes.c_int64), ("bytes_qz", ctypes.c_int64)]


class pf_kernel_info(ctypes.Structure):
    _fields_ = [("tile_x", ctypes.c_int32), ("tile_y", ctypes.c_int32), ("z_chunk", ctypes.c_int32),
                ("threads_per_cta", ctypes.c_int32), ("ctas", ctypes.c_int32), ("regs_per_thread", ctypes.c_int32),
                ("smem_bytes", ctypes.c_int32), ("ctas_per_sm", ctypes.c_int32),
                ("algorithmic_bytes_per_iteration", ctypes.c_int64), ("device_bytes", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("staged", ctypes.c_int32), ("work_items", ctypes.c_int32),
                ("model", ctypes.c_int32), ("flow_nodes", ctypes.c_int32), ("cluster", ctypes.c_int32),
                ("phase1_ctas", ctypes.c_int32), ("tblock", ctypes.c_int32)]


_vp = ctypes.c_void_p
_P = ctypes.POINTER
_sig = {
    "pf_create": (ctypes.c_int, [_P(pf_dims), _P(pf_graph), _P(ctypes.c_void_p), _P(pf_smoothness), _P(pf_config),
                                 _P(pf_slab), _P(ctypes.c_void_p)]),
    "pf_reset": (ctypes.c_int, [_vp]),
    "pf_set_step": (ctypes.c_int, [_vp, ctypes.c_float, ctypes.c_float]),
    "pf_iterate": (ctypes.c_int, [_vp, ctypes.c_int32, _P(ctypes.c_float)]),
    "pf_iterate_phase": (ctypes.c_int, [_vp, ctypes.c_int32, _P(ctypes.c_float)]),
    "pf_run": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.c_float, _P(ctypes.c_int32), _P(ctypes.c_float)]),
    "pf_get_labeling": (ctypes.c_int, [_vp, _vp, _vp]),
    "pf_get_flows": (ctypes.c_int, [_vp, _vp]),
    "pf_get_state": (ctypes.c_int, [_vp, _vp, _vp]),
    "pf_set_state": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int32]),
    "pf_get_node_labeling": (ctypes.c_int, [_vp, ctypes.c_int32, _vp]),
    "pf_get_energy": (ctypes.c_int, [_vp, _P(ctypes.c_double), _P(ctypes.c_double)]),
    "pf_iterations": (ctypes.c_int, [_vp, _P(ctypes.c_int64)]),
    "pf_set_stream": (ctypes.c_int, [_vp, _vp]),
    "pf_set_reserved_sms": (ctypes.c_int, [_vp, ctypes.c_int32]),
    "pf_halo_regions": (ctypes.c_int, [_vp, _P(pf_halo)]),
    "pf_exchange_local": (ctypes.c_int, [_P(ctypes.c_void_p), ctypes.c_int32]),
    "pf_link_slabs": (ctypes.c_int, [_P(ctypes.c_void_p), ctypes.c_int32]),
    "pf_ipc_export": (ctypes.c_int, [_vp, _P(pf_ipc_slab)]),
    "pf_ipc_link": (ctypes.c_int, [_vp, _P(pf_ipc_slab), _P(pf_ipc_slab)]),
    "pf_ipc_step": (ctypes.c_int, [_vp, _P(ctypes.c_float)]),
    "pf_iterate_linked": (ctypes.c_int, [_P(ctypes.c_void_p), ctypes.c_int32, ctypes.c_int32, _P(ctypes.c_float)]),
    "pf_get_kernel_info": (ctypes.c_int, [_vp, _P(pf_kernel_info)]),
    "pf_destroy": (None, [_vp]),
    "pf_last_error": (ctypes.c_char_p, []),
    "pf_version": (ctypes.c_char_p, []),
}
for _name, (_res, _args) in _sig.items():
    if "PF_LIB" in os.environ and not hasattr(_lib, _name):
        continue   # an older build selected for A/B timing (tools/ab.py) may lack newer entry points
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class PFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(st: int):
    if st != PF_OK:
        raise PFError(st, _lib.pf_last_error().decode())


def _ptr(a, dtype=None, numel: Optional[int] = None, what: str = "array") -> int:
    """Raw address of a C-contiguous numpy array (host) or torch tensor (host or CUDA), validated: the
    library reads / writes exactly `numel` elements of `dtype` there, so a wrong dtype, size or layout is
    a ValueError here instead of silently wrong data or an out-of-bounds write in the library."""
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError(f"{what}: numpy arrays must be C-contiguous")
        if dtype is not None and a.dtype != np.dtype(dtype):
            raise ValueError(f"{what}: dtype {a.dtype}, expected {np.dtype(dtype)}")
        if numel is not None and a.size != numel:
            raise ValueError(f"{what}: {a.size} elements, expected {numel}")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError(f"{what}: tensors must be contiguous")
        if dtype is not None:
            import torch
            want = {np.dtype(np.float32): torch.float32, np.dtype(np.uint8): torch.uint8}[np.dtype(dtype)]
            if a.dtype != want:
                raise ValueError(f"{what}: dtype {a.dtype}, expected {want}")
        if numel is not None and a.numel() != numel:
            raise ValueError(f"{what}: {a.numel()} elements, expected {numel}")
        return a.data_ptr()
    raise TypeError(f"{what}: {type(a)} is neither a numpy array nor a tensor")


# geometry per handle, registered by pf_create (V_local, NL, num_nodes, ndim): the sizes the validated
# output / state pointers must have
_GEOM = {}


def pf_version() -> str:
    return _lib.pf_version().decode()


def pf_last_error() -> str:
    return _lib.pf_last_error().decode()


def pf_create(dims: Sequence[int], ndim: int, num_nodes: int, parent, child, weight, D: Sequence, s_kind: int, s_scalars=None,
              s_fields: Optional[Sequence] = None, c: float = 0.25, tau: float = 0.1, cap: int = PF_CAP_L2,
              shift: int = PF_SHIFT_MIN, check_every: int = 10, slab: Optional[Sequence[int]] = None,
              d_bf16: bool = False, method: int = 0, ipc: bool = False, u_half: bool = False,
              tblock: int = 0) -> int:
    """pf_create.  dims = (nx, ny, nz) global.  D: one float32 volume per end label (node-id order)
    covering the slab plus the plane above it.  Returns the opaque solver handle."""
    nx, ny, nz = [int(v) for v in dims]
    d = pf_dims(ndim, nx, ny, nz)
    par = np.ascontiguousarray(parent, dtype=np.int32)
    chi = np.ascontiguousarray(child, dtype=np.int32)
    w = np.ascontiguousarray(weight, dtype=np.float32)
    g = pf_graph(int(num_nodes), len(par),
                 par.ctypes.data_as(_P(ctypes.c_int32)), chi.ctypes.data_as(_P(ctypes.c_int32)),
                 w.ctypes.data_as(_P(ctypes.c_float)))
    z0, z1 = (0, nz) if slab is None else (int(slab[0]), int(slab[1]))
    nD = nx * ny * (min(z1 + 1, nz) - z0)
    Dp = (ctypes.c_void_p * len(D))(*[_ptr(x, np.float32, nD, f"D[{i}]") for i, x in enumerate(D)])
    keep = [par, chi, w, Dp]
    sc = None
    fp = None
    if s_scalars is not None:
        sc = np.ascontiguousarray(s_scalars, dtype=np.float32)
        keep.append(sc)
    if s_fields is not None:
        fp = (ctypes.c_void_p * len(s_fields))(*[_ptr(x, np.float32, nx * ny * (z1 - z0), f"S field {i}")
                                                 for i, x in enumerate(s_fields)])
        keep.append(fp)
    sm = pf_smoothness(s_kind, sc.ctypes.data_as(_P(ctypes.c_float)) if sc is not None else None,
                       ctypes.cast(fp, _P(ctypes.c_void_p)) if fp is not None else None)
    cfg = pf_config(c, tau, cap, shift, check_every, 1 if d_bf16 else 0, 1 if ipc else 0, int(method),
                    1 if u_half else 0, int(tblock))
    sl = pf_slab(int(slab[0]), int(slab[1])) if slab is not None else None
    out = ctypes.c_void_p()
    _check(_lib.pf_create(ctypes.byref(d), ctypes.byref(g), ctypes.cast(Dp, _P(ctypes.c_void_p)), ctypes.byref(sm),
                          ctypes.byref(cfg), ctypes.byref(sl) if sl is not None else None, ctypes.byref(out)))
    _GEOM[out.value] = (nx * ny * (z1 - z0), len(D), int(num_nodes), int(ndim))
    return out.value


def pf_reset(s: int):
    _check(_lib.pf_reset(s))


def pf_set_step(s: int, c: float, tau: float):
    _check(_lib.pf_set_step(s, float(c), float(tau)))


def pf_iterate(s: int, n: int, want_residual: bool = False) -> Optional[float]:
    r = ctypes.c_float(-1.0)
    _check(_lib.pf_iterate(s, int(n), ctypes.byref(r) if want_residual else None))
    return float(r.value) if want_residual else None


def pf_run(s: int, max_iters: int, tol: float):
    """Iterate until the check-iteration residual <= tol or max_iters; returns (iterations, residual)."""
    n = ctypes.c_int32(0)
    r = ctypes.c_float(-1.0)
    _check(_lib.pf_run(s, int(max_iters), float(tol), ctypes.byref(n), ctypes.byref(r)))
    return int(n.value), float(r.value)


def pf_iterate_phase(s: int, phase: int, want_residual: bool = False) -> Optional[float]:
    r = ctypes.c_float(-1.0)
    _check(_lib.pf_iterate_phase(s, int(phase), ctypes.byref(r) if want_residual else None))
    return float(r.value) if want_residual else None


def _sizes(s: int):
    V, NL, nn, nd = _GEOM[s]
    return V, NL, (nn - 1) * nd * V


def pf_get_labeling(s: int, u=None, argmax=None):
    V, NL, _ = _sizes(s)
    _check(_lib.pf_get_labeling(s, _ptr(u, np.float32, NL * V, "u") if u is not None else None,
                                _ptr(argmax, np.uint8, V, "argmax") if argmax is not None else None))


def pf_get_flows(s: int, q):
    _check(_lib.pf_get_flows(s, _ptr(q, np.float32, _sizes(s)[2], "q")))


def pf_get_state(s: int, u_log2=None, q=None):
    """The exact resumable state: lambda = log2 u [NL][z][y][x] and q (see pf.h)."""
    V, NL, nq = _sizes(s)
    _check(_lib.pf_get_state(s, _ptr(u_log2, np.float32, NL * V, "u_log2") if u_log2 is not None else None,
                             _ptr(q, np.float32, nq, "q") if q is not None else None))


def pf_set_state(s: int, u, q, iterations: int, u_is_log2: bool = True):
    """u: lambda = log2 u as pf_get_state returns it (u_is_log2) or the labeling u itself."""
    V, NL, nq = _sizes(s)
    _check(_lib.pf_set_state(s, None if u is None else _ptr(u, np.float32, NL * V, "u"),
                             None if q is None else _ptr(q, np.float32, nq, "q"), int(iterations),
                             1 if u_is_log2 else 0))


def pf_get_node_labeling(s: int, node: int, out):
    _check(_lib.pf_get_node_labeling(s, int(node), _ptr(out, np.float32, _sizes(s)[0], "u_node")))


def pf_get_energy(s: int):
    e, f = ctypes.c_double(), ctypes.c_double()
    _check(_lib.pf_get_energy(s, ctypes.byref(e), ctypes.byref(f)))
    return e.value, f.value


def pf_iterations(s: int) -> int:
    n = ctypes.c_int64()
    _check(_lib.pf_iterations(s, ctypes.byref(n)))
    return n.value


def pf_set_stream(s: int, stream_ptr: int):
    _check(_lib.pf_set_stream(s, stream_ptr))


def pf_set_reserved_sms(s: int, sms: int):
    """Leave `sms` SMs free during pf_iterate_phase(1) launches (a concurrent exchange kernel can run)."""
    _check(_lib.pf_set_reserved_sms(s, int(sms)))


def pf_halo_regions(s: int) -> pf_halo:
    h = pf_halo()
    _check(_lib.pf_halo_regions(s, ctypes.byref(h)))
    return h


def pf_exchange_local(solvers: Sequence[int]):
    arr = (ctypes.c_void_p * len(solvers))(*solvers)
    _check(_lib.pf_exchange_local(ctypes.cast(arr, _P(ctypes.c_void_p)), len(solvers)))


def pf_link_slabs(solvers: Sequence[int]):
    arr = (ctypes.c_void_p * len(solvers))(*solvers)
    _check(_lib.pf_link_slabs(ctypes.cast(arr, _P(ctypes.c_void_p)), len(solvers)))


def pf_iterate_linked(solvers: Sequence[int], iters: int, want_residual: bool = False) -> Optional[float]:
    arr = (ctypes.c_void_p * len(solvers))(*solvers)
    r = ctypes.c_float(-1.0)
    _check(_lib.pf_iterate_linked(ctypes.cast(arr, _P(ctypes.c_void_p)), len(solvers), int(iters),
                                  ctypes.byref(r) if want_residual else None))
    return float(r.value) if want_residual else None


def pf_ipc_export(s: int) -> bytes:
    """The slab's IPC blob (pf_ipc_slab) as bytes, to be sent to the neighbouring ranks."""
    out = pf_ipc_slab()
    _check(_lib.pf_ipc_export(s, ctypes.byref(out)))
    return bytes(out)


def pf_ipc_link(s: int, below: Optional[bytes], above: Optional[bytes]):
    b = pf_ipc_slab.from_buffer_copy(below) if below is not None else None
    a = pf_ipc_slab.from_buffer_copy(above) if above is not None else None
    _check(_lib.pf_ipc_link(s, ctypes.byref(b) if b is not None else None, ctypes.byref(a) if a is not None else None))


def pf_ipc_step(s: int, want_residual: bool = False) -> Optional[float]:
    r = ctypes.c_float(-1.0)
    _check(_lib.pf_ipc_step(s, ctypes.byref(r) if want_residual else None))
    return float(r.value) if want_residual else None


def pf_get_kernel_info(s: int) -> dict:
    k = pf_kernel_info()
    _check(_lib.pf_get_kernel_info(s, ctypes.byref(k)))
    return {f: getattr(k, f) for f, _ in pf_kernel_info._fields_}


def pf_destroy(s: int):
    _GEOM.pop(s, None)
    _lib.pf_destroy(s)


from .solver import Solver, SlabSet  # noqa: E402  (convenience layer, still marshalling only)
