#!/usr/bin/env python
"""bench.py -- throughput of the pseudo-flow hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], "C2"): 3D Potts, 256^3 voxels, 8 labels, 300 iterations, seeded
synthetic ellipsoid phantom.  One STEP = one pass of the whole hot path over the volume: state
init (row a0) + 300 fused iterations with the residual check every 10 (a1-a8) + thresholded
labeling (a9).  With N GPUs (torchrun) every rank owns a 256^3 z-slab of a 256x256x(256N) volume
of the same recipe and exchanges halo planes every iteration (weak scaling).

value = voxel-label-iterations of all ranks / (max over ranks of the CUDA-event time of K steps),
in Gvoxel-label-iterations/s.  The state (4.9 GB) is far larger than L2 (126 MB), so no L2 flush
is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gvoxel-label-iterations/s and achieved HBM GB/s vs peak at 1/2/4/8 B200"
UNIT = "Gvoxel-label-iterations/s"
FALLBACK_HBM = 6650.0


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.dev), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r.split(",") for r in (self.out or "").strip().splitlines() if r.count(",") >= 5]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[2 + i] and "Not" not in r[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _workload(world):
    import phantoms as P
    base = P.config("C2")
    cfg = base.resized(base.nx, base.ny, base.nz * world, name="C2" if world == 1 else f"C2x{world}")
    return base, cfg


def _inputs_for_rank(cfg, rank, world, pinned=False):
    import numpy as np
    import phantoms as P
    from paper_1501_07844_b200.solver import slab_bounds
    z0, z1 = slab_bounds(cfg.nz, world)[rank]
    zt = min(z1 + 1, cfg.nz)
    inp = P.generate(cfg, (z0, zt, 0, cfg.ny, 0, cfg.nx))
    D = [np.ascontiguousarray(inp.D[l]) for l in range(inp.D.shape[0])]
    S = np.ascontiguousarray(inp.s_field[: z1 - z0])
    if pinned:
        import torch
        D = [torch.from_numpy(d).pin_memory() for d in D]
        S = torch.from_numpy(S).pin_memory()
    return inp.graph, (z0, z1), D, S


def cpu_oracle_rate(iters: int, planes: int = 64):
    """The oracle (as it stands) on a bounded sample: `iters` iterations of a 256x256x`planes` window of C2."""
    import numpy as np
    import oracle as O
    import phantoms as P
    cfg = P.config("C2")
    inp = P.generate(cfg, (0, planes, 0, cfg.ny, 0, cfg.nx))
    D = np.ascontiguousarray(inp.D, dtype=np.float64)
    S = np.empty((8,) + inp.shape)
    S[:] = inp.s_field
    u, q = O.init_state(8, 8, inp.shape, 3)
    t0 = time.perf_counter()
    O.potts_iterate(D, S, u, q, 3, cfg.c, cfg.tau, iters)
    dt = time.perf_counter() - t0
    vl = inp.D.size * iters
    return vl / dt / 1e9, dt, f"{iters} oracle iteration(s) of a 256x256x{planes} window of C2 (K=8), fp64, 1 thread"


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle timed on this box's host cores (rank 0 only)."""
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_oracle_rate(1)
    t_tot, vl_rate = 0.0, []
    for _ in range(args.steps):
        r, dt, sample = cpu_oracle_rate(1)
        t_tot += dt
        vl_rate.append(r)
    value = sum(vl_rate) / len(vl_rate)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t_tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C2: 3D Potts 256^3, K=8 (oracle, bounded sample per step)",
                       "sample_per_step": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1501_07844_b200 as pf
    from paper_1501_07844_b200.dist import DistSolver

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    base, cfg = _workload(world)
    iters = args.iters or base.iters
    g, slab, D, S = _inputs_for_rank(cfg, rank, world)

    ipc = args.transport == "ipc" and world > 1

    def make(slab_):
        return pf.Solver((cfg.nx, cfg.ny, cfg.nz), 3, (g.num_nodes, g.parent, g.child, g.weight), D, s_shared=S,
                         c=cfg.c, tau=cfg.tau, check_every=10, slab=slab_, ipc=ipc)

    ds = DistSolver(make, cfg.nz, rank, world, dev, transport=args.transport)
    s = ds.solver
    stream = torch.cuda.current_stream(dev)
    V = cfg.nx * cfg.ny * (slab[1] - slab[0])
    NL = len(D)
    labels = torch.empty((slab[1] - slab[0], cfg.ny, cfg.nx), dtype=torch.uint8, device=dev)

    def step(evs=None):
        ds.reset()
        if evs is not None:
            evs[0].record(stream)
        ds.iterate(iters)
        if evs is not None:
            evs[1].record(stream)
        pf.pf_get_labeling(s.h, None, labels)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    kevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = s.kernel_info()["kernel_launches"]
    with ClockSampler(local_rank) as clk:
        time.sleep(0.25)
        t_start.record(stream)
        for k in range(args.steps):
            step(kevs[k])
        t_end.record(stream)
        torch.cuda.synchronize()
    launches = s.kernel_info()["kernel_launches"] - launches0
    if world > 1:
        dist.barrier()
    ms = t_start.elapsed_time(t_end)
    iter_ms = sum(a.elapsed_time(b) for a, b in kevs)
    t = torch.tensor([ms, iter_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, iter_ms = float(t[0]), float(t[1])
    info = s.kernel_info()
    vl_total = V * world * NL * iters * args.steps
    value = vl_total / (ms / 1e3) / 1e9
    # roofline of the dominant kernel (pf_iter_staged): algorithmic bytes per launch / mean launch time
    per_launch_ms = iter_ms / (iters * args.steps)
    alg_bytes = info["algorithmic_bytes_per_iteration"]
    achieved = alg_bytes / (per_launch_ms / 1e3) / 1e9
    peak, peak_src = _peaks()
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            tj = json.load(fh)
        if tj.get("workload") == cfg.name and tj.get("kernel_config") == [info["tile_x"], info["tile_y"],
                                                                           info["z_chunk"]]:
            traffic = tj.get("dram_bytes_per_launch")
    # ------------------------------------------------------------ end to end through the public API
    e2e = None
    if not args.no_e2e:
        gH, slabH, DH, SH = _inputs_for_rank(cfg, rank, world, pinned=True)
        u_host = torch.empty((NL, slab[1] - slab[0], cfg.ny, cfg.nx), dtype=torch.float32).pin_memory()
        lab_host = torch.empty((slab[1] - slab[0], cfg.ny, cfg.nx), dtype=torch.uint8).pin_memory()
        h2d = sum(d.numel() * 4 for d in DH) + SH.numel() * 4
        d2h = u_host.numel() * 4 + lab_host.numel()

        def e2e_step():
            def mk(slab_):
                return pf.Solver((cfg.nx, cfg.ny, cfg.nz), 3, (gH.num_nodes, gH.parent, gH.child, gH.weight), DH,
                                 s_shared=SH, c=cfg.c, tau=cfg.tau, check_every=10, slab=slab_, ipc=ipc)
            if world == 1:   # the single-GPU user path: one Solver on its own stream
                sv = mk(None)
                sv.iterate(iters)
                sv.labeling(u_host, lab_host)
                sv.close()
                return
            d = DistSolver(mk, cfg.nz, rank, world, dev, transport=args.transport)
            d.iterate(iters)
            d.solver.labeling(u_host, lab_host)
            d.close()

        e2e_step()
        torch.cuda.synchronize()
        ne = max(1, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ne):
            e2e_step()
        torch.cuda.synchronize()
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": V * world * NL * iters * ne / float(te[0]) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": ne,
               "path": "pf_create(pinned host D,S) + pf_iterate(300) + pf_get_labeling(pinned host u, argmax) + "
                       "pf_destroy, wall clock"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, dt, sample = cpu_oracle_rate(4)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample, "seconds": round(dt, 2)}
    ds.close()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name + (": 3D Potts 256^3, K=8, 300 iterations" if world == 1 else
                                                f": 3D Potts 256x256x{cfg.nz} (256^3 z-slab per GPU), K=8, "
                                                f"{iters} iterations, halo exchange: " +
                                                ("fused CUDA-IPC peer stores" if ipc else "NCCL P2P, overlapped" if dist.get_backend() == "nccl" else f"{dist.get_backend()} host-staged (validation only, not a measurement)")),
                       "voxels_per_gpu": V, "labels": NL, "iterations_per_step": iters, "residual_check_every": 10,
                       "l2": "no flush: per-iteration state 4.9 GB/GPU >> 126 MB L2",
                       "kernel": {k: info[k] for k in ("tile_x", "tile_y", "z_chunk", "threads_per_cta", "ctas",
                                                        "regs_per_thread", "smem_bytes", "ctas_per_sm")}},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "pf_iter_staged" if info["staged"] else "pf_iter_kernel",
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "mean_launch_ms": per_launch_ms},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--iters", type=int, default=0, help="override iterations per step (default: config's 300)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--transport", choices=["nccl", "ipc"], default="nccl",
                    help="N > 1: halo exchange by NCCL P2P overlapped with the interior (default), or fused into "
                         "the kernels as CUDA-IPC peer stores (pf_ipc_*)")
    args = ap.parse_args()
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    # validation only (never for a reported number): PF_BENCH_BACKEND=gloo with PF_BENCH_ONE_GPU=1 runs the
    # N-rank code path as N processes on cuda:0 (host-staged halo exchange, see dist.halo_exchange)
    backend = os.environ.get("PF_BENCH_BACKEND", "nccl")
    if os.environ.get("PF_BENCH_ONE_GPU") == "1":
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
