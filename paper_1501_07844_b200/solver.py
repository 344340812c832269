"""Convenience wrappers over the C-ABI (marshalling only; all compute is in libpf.so)."""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from . import (PF_CAP_L2, PF_SHIFT_MIN, PF_S_FIELD_PER_NODE, PF_S_SCALAR_PER_NODE, PF_S_SCALED_FIELD,
               PF_S_SHARED_FIELD,
               pf_create, pf_destroy, pf_exchange_local, pf_iterate_linked, pf_link_slabs, pf_get_energy, pf_get_flows, pf_get_kernel_info,
               pf_get_labeling, pf_get_node_labeling, pf_get_state, pf_halo_regions, pf_iterate, pf_iterate_phase, pf_iterations, pf_reset, pf_run,
               pf_set_reserved_sms, pf_set_state, pf_set_step,
               pf_set_stream)


class Solver:
    """One pseudo-flow solver (one device, one z-slab or the whole volume).

    graph = (num_nodes, parent, child, weight) with node 0 the source;
    D = one float32 [z][y][x] volume per end label (numpy or CUDA tensor) covering the
    slab plus the plane above it; capacities: exactly one of `s_scalars` ([num_nodes]),
    `s_shared` (one volume), `s_fields` (one volume per non-source node) or `s_scaled` =
    (factors [num_nodes], volume): S_v(x) = factors[v] * volume(x).
    """

    def __init__(self, dims: Sequence[int], ndim: int, graph, D: Sequence, *, s_scalars=None, s_shared=None,
                 s_fields=None, s_scaled=None, c: float = 0.25, tau: float = 0.1, cap: int = PF_CAP_L2,
                 shift: int = PF_SHIFT_MIN, check_every: int = 10, slab: Optional[Sequence[int]] = None,
                 d_bf16: bool = False, method: int = 0, ipc: bool = False, u_half: bool = False,
                 tblock: int = 0):
        num_nodes, parent, child, weight = graph
        self.dims = tuple(int(v) for v in dims)
        self.ndim = ndim
        self.num_nodes = int(num_nodes)
        self.NL = len(D)
        self.slab = (0, self.dims[2]) if slab is None else (int(slab[0]), int(slab[1]))
        self.check_every = int(check_every)
        if s_scaled is not None:
            kind, s_scalars, fields = PF_S_SCALED_FIELD, s_scaled[0], [s_scaled[1]]
        elif s_scalars is not None:
            kind, fields = PF_S_SCALAR_PER_NODE, None
        elif s_shared is not None:
            kind, fields = PF_S_SHARED_FIELD, [s_shared]
        else:
            kind, fields = PF_S_FIELD_PER_NODE, list(s_fields)
        self.h = pf_create(self.dims, ndim, num_nodes, parent, child, weight, list(D), kind, s_scalars, fields, c, tau, cap,
                           shift, check_every, slab, d_bf16, method, ipc, u_half, tblock)

    # ---------------------------------------------------------------- C-ABI calls
    @property
    def nz_local(self) -> int:
        return self.slab[1] - self.slab[0]

    @property
    def shape(self):
        return (self.nz_local, self.dims[1], self.dims[0])

    def reset(self):
        pf_reset(self.h)

    def iterate(self, n: int, residual: bool = False):
        return pf_iterate(self.h, n, residual)

    def set_step(self, c: float, tau: float):
        """New step constants for the following iterations (c-annealing); the state is kept."""
        pf_set_step(self.h, c, tau)

    def run(self, max_iters: int, tol: float):
        """Iterate until converged (residual <= tol at a check iteration) or max_iters: (iterations, residual)."""
        return pf_run(self.h, max_iters, tol)

    def iterate_phase(self, phase: int, residual: bool = False):
        """One iteration in two launches (boundary planes, then the rest); see pf_iterate_phase."""
        return pf_iterate_phase(self.h, phase, residual)

    def set_stream(self, stream_ptr: int):
        pf_set_stream(self.h, stream_ptr)

    def set_reserved_sms(self, sms: int):
        """SMs a pf_iterate_phase(1) launch leaves free for a concurrent exchange kernel (pf_set_reserved_sms)."""
        pf_set_reserved_sms(self.h, sms)

    def labeling(self, u_out=None, argmax_out=None):
        """Return (u [NL][z][y][x] float32, argmax [z][y][x] uint8) as numpy unless outputs are given."""
        ret_u = u_out is None
        ret_a = argmax_out is None
        if u_out is None:
            u_out = np.empty((self.NL,) + self.shape, dtype=np.float32)
        if argmax_out is None:
            argmax_out = np.empty(self.shape, dtype=np.uint8)
        pf_get_labeling(self.h, u_out, argmax_out)
        return u_out, argmax_out

    def node_labeling(self, node: int, out=None):
        """u_v = sum_B W_(v,B) u_B of any graph node (intermediate labels on demand), [z][y][x] float32."""
        if out is None:
            out = np.empty(self.shape, dtype=np.float32)
        pf_get_node_labeling(self.h, node, out)
        return out

    def flows(self):
        q = np.empty((self.num_nodes - 1, self.ndim) + self.shape, dtype=np.float32)
        pf_get_flows(self.h, q)
        return q

    def energy(self):
        return pf_get_energy(self.h)

    # ---------------------------------------------------------------- checkpoint / resume
    def state(self):
        """(lambda = log2 u, q, iterations): the exact resumable state of the owned slab (pf_get_state)."""
        lam = np.empty((self.NL,) + self.shape, dtype=np.float32)
        q = np.empty((self.num_nodes - 1, self.ndim) + self.shape, dtype=np.float32)
        pf_get_state(self.h, lam, q)
        return lam, q, self.iterations()

    def set_state(self, u, q, iterations: int, u_is_log2: bool = True):
        """Restore a state from state() (pf_set_state; u = lambda = log2 u), or start from a labeling u
        (u_is_log2=False); slab solvers then need a halo exchange."""
        pf_set_state(self.h, np.ascontiguousarray(u) if isinstance(u, np.ndarray) else u,
                     np.ascontiguousarray(q) if isinstance(q, np.ndarray) else q, iterations, u_is_log2)

    def save(self, path: str, c: Optional[float] = None, tau: Optional[float] = None):
        """Checkpoint to one .npz: lambda = log2 u, q (raw float32), the iteration count and the geometry it
        belongs to (plus the current c, tau if given: they are configuration, not state)."""
        u, q, it = self.state()
        meta = {"dims": self.dims, "ndim": self.ndim, "num_nodes": self.num_nodes, "labels": self.NL,
                "slab": self.slab, "iterations": it, "c": c, "tau": tau}
        np.savez(path, u=u, q=q, meta=np.frombuffer(repr(meta).encode(), dtype=np.uint8))

    def load(self, path: str):
        """Resume from save(): checks the geometry, restores u, q and the iteration count; returns the
        saved (c, tau) (None where not saved) so a schedule can continue with pf_set_step."""
        import ast
        z = np.load(path)
        meta = ast.literal_eval(bytes(z["meta"]).decode())
        mine = {"dims": self.dims, "ndim": self.ndim, "num_nodes": self.num_nodes, "labels": self.NL,
                "slab": self.slab}
        for k, v in mine.items():
            if (tuple(meta[k]) if isinstance(v, tuple) else meta[k]) != v:
                raise ValueError(f"checkpoint {k} = {meta[k]} does not match this solver's {v}")
        self.set_state(z["u"], z["q"], meta["iterations"])
        return meta.get("c"), meta.get("tau")

    def iterations(self) -> int:
        return pf_iterations(self.h)

    def halo(self):
        return pf_halo_regions(self.h)

    def kernel_info(self) -> dict:
        return pf_get_kernel_info(self.h)

    def close(self):
        if self.h:
            pf_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def slab_bounds(nz: int, parts: int) -> List[tuple]:
    """z-slabs of ceil(nz/parts) planes; the last may be shorter."""
    h = -(-nz // parts)
    out = []
    for r in range(parts):
        z0, z1 = r * h, min(nz, (r + 1) * h)
        if z0 < z1:
            out.append((z0, z1))
    return out


class SlabSet:
    """A volume split into consecutive z-slab solvers driven from one process (one or several
    devices); halos are exchanged by pf_exchange_local after every iteration."""

    def __init__(self, solvers: Sequence[Solver], phased: bool = False, fused: bool = False):
        """phased: every iteration as pf_iterate_phase 0 + 1 (the NCCL multi-GPU schedule); fused: link the
        slabs (pf_link_slabs) so the iteration kernels store their boundary planes straight into the
        neighbours' halos (peer memory) -- no exchange step."""
        self.solvers = list(solvers)
        self.handles = [s.h for s in self.solvers]
        self.phased = phased
        self.fused = fused and len(self.solvers) > 1
        if self.fused:
            pf_link_slabs(self.handles)

    def iterate(self, n: int, residual: bool = False):
        if self.fused:
            return pf_iterate_linked(self.handles, n, residual)
        r = None
        for t in range(n):
            last = residual and t == n - 1
            if self.phased:
                for s in self.solvers:
                    s.iterate_phase(0)
                vals = [s.iterate_phase(1, last) for s in self.solvers]
            else:
                vals = [s.iterate(1, last) for s in self.solvers]
            pf_exchange_local(self.handles)
            if last:
                r = max(vals)
        return r

    def exchange(self):
        pf_exchange_local(self.handles)

    def state(self):
        """(lambda = log2 u, q, iterations) of the whole volume (slabs concatenated along z)."""
        st = [s.state() for s in self.solvers]
        return (np.concatenate([x[0] for x in st], axis=1), np.concatenate([x[1] for x in st], axis=2),
                self.solvers[0].iterations())

    def set_state(self, u, q, iterations: int):
        """Restore a whole-volume state: every slab takes its planes, then one halo exchange."""
        for sv in self.solvers:
            z0, z1 = sv.slab
            sv.set_state(np.ascontiguousarray(u[:, z0:z1]), np.ascontiguousarray(q[:, :, z0:z1]), iterations)
        pf_exchange_local(self.handles)

    def labeling(self):
        us, ams = zip(*[s.labeling() for s in self.solvers])
        return np.concatenate(us, axis=1), np.concatenate(ams, axis=0)

    def flows(self):
        return np.concatenate([s.flows() for s in self.solvers], axis=2)

    def energy(self):
        es = [s.energy() for s in self.solvers]
        return sum(e for e, _ in es), sum(f for _, f in es)

    def close(self):
        for s in self.solvers:
            s.close()
