"""Multi-GPU z-slab driver: one process per GPU, halo planes exchanged with torch.distributed P2P.

Row e of the hot-path scope: the volume is split into z-slabs of
ceil(nz/P) planes; after every iteration rank r sends its first-plane u and q to r-1 and its
last-plane q^z to r+1 (pf_halo_regions names the device ranges).  The exchange rides on the
process group (NCCL over NVLink on a GPU box, gloo on CPU for the host-side tests).

Overlap (BASELINE.json north_star: "halo exchange ... overlapped with interior compute"): every
iteration is issued as pf_iterate_phase 0 (the boundary planes only) and phase 1 (the rest) on the
solver's stream S; the exchange is posted on a communication stream C that waits for an event
recorded between the two phases, so NCCL moves the boundary planes while phase 1 computes the
interior.  S waits for the exchange before the next phase 0 (which reads the received halos).
The received planes land in halo planes of the new state that phase 1 neither reads nor writes.

The persistent interior launch would otherwise hold every SM (one ~216 KB CTA each) until it drains, so
the exchange kernel could not start before it: with NCCL the solver reserves `reserve_sms` SMs for it
(pf_set_reserved_sms; the work-item queue finishes the same items on the smaller grid, bitwise equal).

transport="ipc" (solvers created with ipc=True): no exchange step at all -- the iteration kernels store
their boundary planes straight into the neighbours' halo planes through CUDA-IPC-mapped peer memory
(pf_ipc_*), ordered ON THE DEVICE: each step's stream waits (cuStreamWaitValue32) for the neighbours'
progress words and announces its own (cuStreamWriteValue32) -- no host barrier per iteration.

NVTX ranges (nsys): "pf boundary" / "pf interior" (the library), "pf halo exchange" (here), "pf ipc step",
"pf check (residual read)".
"""
from __future__ import annotations

from typing import Dict, Optional

import torch
import torch.distributed as dist

from . import pf_ipc_export, pf_ipc_link, pf_ipc_step
from .solver import Solver, slab_bounds


class _CudaBuf:
    """__cuda_array_interface__ view of a raw device range (zero-copy into torch)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes // 4,), "typestr": "<f4", "data": (int(ptr), False),
                                         "version": 3}


def device_view(ptr: int, nbytes: int, device: torch.device) -> torch.Tensor:
    return torch.as_tensor(_CudaBuf(ptr, nbytes), device=device)


class _StreamWork:
    """Work handle of a host-staged exchange: wait() orders the caller's current stream after it."""

    def __init__(self, ev):
        self.ev = ev

    def wait(self):
        torch.cuda.current_stream().wait_event(self.ev)


def halo_exchange(regions: Dict[str, Optional[torch.Tensor]], rank: int, world: int, group=None, wait: bool = True):
    """Exchange one iteration's halo planes.  regions: send_down_u, send_down_q, recv_up_u, recv_up_q,
    send_up_qz, recv_down_qz (None where the neighbour does not exist).  Per peer pair the messages
    are posted in the same order on both sides (u, then q downward; q^z upward).  wait=False returns
    the work handles (their wait() orders the caller's current stream after the transfer).
    Device regions over a backend without device transport (gloo: multi-process tests on one GPU)
    are staged through host memory on the current stream; NCCL moves them device to device."""
    if dist.get_backend(group) != "nccl" and any(v is not None and v.is_cuda for v in regions.values()):
        host = {k: (v.cpu() if k.startswith("send") else torch.empty(v.shape, dtype=v.dtype))
                for k, v in regions.items() if v is not None}
        halo_exchange({k: host.get(k) for k in regions}, rank, world, group, wait=True)
        for k, v in regions.items():
            if v is not None and k.startswith("recv"):
                v.copy_(host[k])
        if wait:
            return []
        ev = torch.cuda.Event()
        ev.record()
        return [_StreamWork(ev)]
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, regions["send_down_u"], rank - 1, group))
        ops.append(dist.P2POp(dist.isend, regions["send_down_q"], rank - 1, group))
        if regions.get("recv_down_qz") is not None:
            ops.append(dist.P2POp(dist.irecv, regions["recv_down_qz"], rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.irecv, regions["recv_up_u"], rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, regions["recv_up_q"], rank + 1, group))
        if regions.get("send_up_qz") is not None:
            ops.append(dist.P2POp(dist.isend, regions["send_up_qz"], rank + 1, group))
    works = dist.batch_isend_irecv(ops) if ops else []
    if wait:
        for w in works:
            w.wait()
        return []
    return works


class DistSolver:
    """The rank's slab solver plus its halo exchange.  `make_solver(slab)` builds the Solver."""

    def __init__(self, make_solver, nz: int, rank: int, world: int, device: torch.device, group=None,
                 transport: str = "nccl", reserve_sms: int = 8):
        self.rank, self.world, self.group = rank, world, group
        self.transport = transport
        self.device = device
        self.bounds = slab_bounds(nz, world)
        assert len(self.bounds) == world, "every rank needs at least one plane"
        self.slab = self.bounds[rank]
        self.solver: Solver = make_solver(self.slab)
        self.cuda = torch.device(device).type == "cuda"
        if self.cuda:
            self.solver.set_stream(torch.cuda.current_stream(device).cuda_stream)
            if transport == "nccl" and world > 1 and reserve_sms > 0:
                self.solver.set_reserved_sms(reserve_sms)   # room for NCCL's P2P kernel during phase 1
        self.host_group = group
        if transport == "ipc" and world > 1:
            # host-only barriers at link and close (a NCCL barrier would queue behind the GPU work)
            if dist.get_backend(group) != "gloo":
                self.host_group = dist.new_group(backend="gloo")
            blobs = [None] * world
            dist.all_gather_object(blobs, pf_ipc_export(self.solver.h), group=group)
            pf_ipc_link(self.solver.h, blobs[rank - 1] if rank > 0 else None,
                        blobs[rank + 1] if rank < world - 1 else None)
            dist.barrier(group=self.host_group)   # every rank has recorded "initial state in place"

    def _regions(self):
        h = self.solver.halo()
        dv = self.device
        return {
            "send_down_u": device_view(h.send_down_u, h.bytes_u, dv) if h.send_down_u else None,
            "send_down_q": device_view(h.send_down_q, h.bytes_q, dv) if h.send_down_q else None,
            "recv_up_u": device_view(h.recv_up_u, h.bytes_u, dv) if h.recv_up_u else None,
            "recv_up_q": device_view(h.recv_up_q, h.bytes_q, dv) if h.recv_up_q else None,
            "send_up_qz": device_view(h.send_up_qz, h.bytes_qz, dv) if h.send_up_qz else None,
            "recv_down_qz": device_view(h.recv_down_qz, h.bytes_qz, dv) if h.recv_down_qz else None,
        }

    def _last_check_index(self, n: int):
        """Index t in [0, n) of the last check iteration of this call (pf_iterate's residual), or None."""
        k = getattr(self.solver, "check_every", 0)
        if k <= 0:
            return None
        it0 = self.solver.iterations()
        t = n - 1 - ((it0 + n) % k)
        return t if t >= 0 else None

    def iterate(self, n: int, residual: bool = False, overlap: bool = True):
        """n iterations with the halo exchange after each.  residual=True: as pf_iterate -- the residual of
        the last check iteration of this call, max over ranks (-1 if there was none)."""
        if self.world == 1:
            return self.solver.iterate(n, residual)
        want = self._last_check_index(n) if residual else None
        r = -1.0 if residual else None
        if self.transport == "ipc":
            # ordered on the device (progress words); the ranks' streams run ahead without host barriers
            for t in range(n):
                val = pf_ipc_step(self.solver.h, t == want)
                if t == want:
                    r = self._max_over_ranks(val)
            return r
        overlap = overlap and self.cuda
        S = torch.cuda.current_stream(self.device) if self.cuda else None
        C = self._comm_stream() if overlap else None
        works = []
        for t in range(n):
            for w in works:      # S waits for the previous exchange (the halos phase 0 reads)
                w.wait()
            works = []
            if overlap:
                self.solver.iterate_phase(0)
                ev = torch.cuda.Event()
                ev.record(S)
                val = self.solver.iterate_phase(1, t == want)
                C.wait_event(ev)
                torch.cuda.nvtx.range_push("pf halo exchange")
                with torch.cuda.stream(C):
                    works = halo_exchange(self._regions(), self.rank, self.world, self.group, wait=False)
                torch.cuda.nvtx.range_pop()
            else:
                val = self.solver.iterate(1, t == want)
                halo_exchange(self._regions(), self.rank, self.world, self.group)
            if t == want:
                r = self._max_over_ranks(val)
        for w in works:
            w.wait()
        return r

    def _reduce_device(self):
        return self.device if dist.get_backend(self.group) == "nccl" else torch.device("cpu")

    def _max_over_ranks(self, val: float) -> float:
        rt = torch.tensor([val], dtype=torch.float64, device=self._reduce_device())
        dist.all_reduce(rt, op=dist.ReduceOp.MAX, group=self.group)
        return float(rt.item())

    def run(self, max_iters: int, tol: float):
        """"while not converged" across the slabs: iterate until the residual of a check iteration, max
        over ranks (all-reduce MAX), is <= tol or max_iters.  Returns (iterations, residual)."""
        k = self.solver.check_every
        if k <= 0:
            raise ValueError("run() needs check_every > 0")
        done, r = 0, -1.0
        while done < max_iters:
            it = self.solver.iterations()
            n = min(k - it % k, max_iters - done)
            rr = self.iterate(n, residual=True)
            done += n
            if (it + n) % k == 0:
                r = rr
                if r <= tol:
                    break
        return done, r

    def energy(self):
        """(primal, dual) of the whole volume: the slabs' fp64 energies summed over ranks (all-reduce SUM).
        The halos must be current (they are after iterate())."""
        e, f = self.solver.energy()
        if self.world == 1:
            return e, f
        t = torch.tensor([e, f], dtype=torch.float64, device=self._reduce_device())
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return float(t[0]), float(t[1])

    # ------------------------------------------------------------ checkpoint / resume (pf_set_state)
    def _rank_path(self, prefix: str) -> str:
        return f"{prefix}.rank{self.rank}of{self.world}.npz"

    def save(self, prefix: str, **meta):
        """Every rank writes its own slab (u, q, iteration count) to <prefix>.rank<r>of<P>.npz."""
        return self.solver.save(self._rank_path(prefix), **meta)

    def load(self, prefix: str):
        """Every rank restores its slab, then the halo planes are refreshed with one exchange (the
        checkpoint holds only owned planes).  Returns the saved (c, tau)."""
        if self.transport == "ipc" and self.world > 1:
            raise NotImplementedError("resume over the IPC transport: the halos are only pushed by iterations")
        out = self.solver.load(self._rank_path(prefix))
        if self.world > 1:
            halo_exchange(self._regions(), self.rank, self.world, self.group)
        return out

    def _comm_stream(self):
        if getattr(self, "_C", None) is None:
            self._C = torch.cuda.Stream(self.device)
        return self._C

    def reset(self):
        self.solver.reset()   # IPC: a step of the device-side protocol (pf_reset), no host barrier

    def close(self):
        if self.transport == "ipc" and self.world > 1:   # no neighbour kernel may still write into our buffers
            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.host_group)
        self.solver.close()
