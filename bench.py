#!/usr/bin/env python
"""bench.py -- throughput of the pseudo-flow hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workloads (BASELINE.json configs; the metric is quoted at 1/2/4/8 B200, its 8-GPU volume C5 does not fit
one GPU, so N = 1 runs the LARGEST single-GPU config):
  * N = 1: C4 -- 3D DAGMF 320^3, 6 end labels + 3 internal nodes (2 leaves shared, weights 0.5/0.5),
    300 iterations.  In the same line, `c5slab`: one 8-GPU rank's share of C5 (768x768x96, K = 16,
    200 iterations) as a standalone volume -- the per-GPU denominator of C5's weak-scaling efficiency
    (SURVEY 8.4.4).
  * N > 1: C5 -- 3D Potts 768^3, K = 16, 200 iterations, z-sharded over the N GPUs (ceil(768/N) planes
    per rank; fits from N = 2), halo planes exchanged every iteration; total work fixed ("strong").
    Without torchrun (no WORLD_SIZE) `--gpus N` re-launches itself under torch.distributed.run.
One STEP = one pass of the whole hot path: state init (row a0) + the configured iterations with the
residual check every 10 (a1-a8) + thresholded labeling (a9).

value = voxel-node-iterations of all ranks / (max over ranks of the CUDA-event time of K steps), in
Gvoxel-label-iterations/s, a "label" being a node that carries a flow (the 9 non-source
nodes of C3/C4; the K end labels of a Potts model).  The state (9.4 GB for C4) is far larger than L2
(126 MB), so no L2 flush is needed between steps.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
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


def source_hash() -> str:
    """Hash of the CUDA sources and the C-ABI header: ties a committed ncu traffic capture to the kernel
    build it measured (a capture of another source state is not reported)."""
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_1501_07844_b200", "csrc")
    files = sorted(f for f in os.listdir(csrc) if f.endswith((".cu", ".cuh", ".h", ".py")))
    for f in files + ["../../include/pf.h"]:
        p = os.path.normpath(os.path.join(csrc, f))
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def _traffic(workload: str, kernel: str):
    """ncu DRAM bytes per launch of `kernel` on `workload` from profiles/ncu_traffic.json, if it was captured
    from the current sources (else None)."""
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(tp):
        return None
    with open(tp) as fh:
        tj = json.load(fh)
    sh = source_hash()
    for e in tj.get("entries", []):
        if e.get("workload") == workload and e.get("src_hash") == sh and kernel in e.get("kernel", ""):
            return e.get("dram_bytes_per_launch")
    return None


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


def workload(world: int, override: str = ""):
    """N = 1: C4 (largest single-GPU config); N > 1: C5 z-sharded.  `override` (--config, experiments and the
    one-GPU code-path test only): C2, C3, C4, C5, C5slab, C5small (192^3, K = 16)."""
    import phantoms as P
    if override == "C5slab":
        return c5slab_config()
    if override == "C5small":
        return P.config("C5").resized(192, 192, 192, name="C5small")
    if override:
        return P.config(override)
    return P.config("C4") if world == 1 else P.config("C5")


def c5slab_config():
    import phantoms as P
    return P.config("C5").resized(768, 768, 96, name="C5slab")


DESCR = {"C2": "C2: 3D Potts 256^3, K=8, 300 iterations",
         "C3": "C3: 3D HMF 256^3, 6 end labels + 3 internal nodes (9 flow nodes), 300 iterations",
         "C5small": "C5small: C5's recipe at 192^3, K=16, 200 iterations (code-path checks only)",
         "C4": "C4: 3D DAGMF 320^3, 6 end labels + 3 internal nodes (9 flow nodes), 300 iterations",
         "C5": "C5: 3D Potts 768^3, K=16, 200 iterations",
         "C5slab": "C5slab: one 8-GPU rank's share of C5 -- 768x768x96, K=16, 200 iterations"}


def inputs_sha256(D, kw) -> str:
    """SHA-256 of the generated inputs of this rank (D volumes, then the capacity field or scalars), logged
    with every result: the phantoms are regenerated from seeds, so equal hashes = equal inputs."""
    import numpy as np
    h = hashlib.sha256()
    for d in D:
        h.update(np.ascontiguousarray(d).view(np.uint8))
    for k in sorted(kw):
        h.update(np.ascontiguousarray(kw[k], dtype=np.float32).view(np.uint8))
    return h.hexdigest()


def inputs_for_rank(cfg, rank, world, pinned=False):
    """(graph, slab, D list, capacity kwargs) of this rank's z-slab (D covers the slab + the plane above)."""
    import numpy as np
    import phantoms as P
    from paper_1501_07844_b200.solver import slab_bounds
    z0, z1 = slab_bounds(cfg.nz, world)[rank]
    zt = min(z1 + 1, cfg.nz)
    inp = P.generate(cfg, (z0, zt, 0, cfg.ny, 0, cfg.nx))
    D = [np.ascontiguousarray(inp.D[l]) for l in range(inp.D.shape[0])]
    if inp.s_kind == "shared_field":
        kw = {"s_shared": np.ascontiguousarray(inp.s_field[: z1 - z0])}
    else:
        kw = {"s_scalars": inp.s_scalars}
    del inp
    if pinned:
        import torch
        D = [torch.from_numpy(d).pin_memory() for d in D]
        kw = {k: (torch.from_numpy(v).pin_memory() if k == "s_shared" else v) for k, v in kw.items()}
    return cfg.graph(), (z0, z1), D, kw


def cpu_oracle_rate(cfg, iters: int, planes: int):
    """The oracle (as it stands: fp64, one thread) on a bounded sample of the workload `cfg`: `iters`
    iterations of an nx x ny x `planes` window of it."""
    import oracle as O
    import phantoms as P
    inp = P.generate(cfg, (0, min(planes, cfg.nz), 0, cfg.ny, 0, cfg.nx))
    t0 = time.perf_counter()
    O.run_inputs(inp, iters)
    dt = time.perf_counter() - t0
    vl = inp.shape[0] * inp.shape[1] * inp.shape[2] * (inp.graph.num_nodes - 1) * iters
    return vl / dt / 1e9, dt, (f"{iters} oracle iteration(s) of a {cfg.nx}x{cfg.ny}x{min(planes, cfg.nz)} window of "
                               f"{cfg.name} ({inp.graph.num_nodes - 1} flow nodes), fp64, 1 thread")


def _cpu_planes(cfg, per_step=False):
    """Window depth for the oracle sample: ~1.5 s per reference-arm step, ~10 s for the cpu_baseline leg."""
    planes = max(1, int(2.0e6 / (cfg.nx * cfg.ny)))   # ~2 M voxels
    return planes if per_step else 4 * planes


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle timed on this box's host cores (rank 0 only), on bounded samples of
    our arm's workload."""
    if rank != 0:
        return
    cfg = workload(world, args.config)
    planes = _cpu_planes(cfg, per_step=True)
    for _ in range(args.warmup):
        cpu_oracle_rate(cfg, 1, planes)
    t_tot, vl_rate = 0.0, []
    for _ in range(args.steps):
        r, dt, sample = cpu_oracle_rate(cfg, 1, planes)
        t_tot += dt
        vl_rate.append(r)
    value = sum(vl_rate) / len(vl_rate)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t_tot / args.steps,
            "higher_is_better": True, "scaling": "weak" if world == 1 else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": DESCR[cfg.name] + " (oracle, bounded sample per step)", "sample_per_step": sample},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _solver_factory(pf, cfg, g, D, kw, ipc=False):
    def make(slab_):
        return pf.Solver((cfg.nx, cfg.ny, cfg.nz), 3, (g.num_nodes, g.parent, g.child, g.weight), D, c=cfg.c,
                         tau=cfg.tau, check_every=10, slab=slab_, ipc=ipc, **kw)
    return make


def time_workload(cfg, rank, world, local_rank, args, iters, steps, warmup, clocks=False):
    """Device time of `steps` whole-hot-path steps of `cfg` on this rank (max over ranks); per-launch time
    of the fused iteration kernel from CUDA events around the iteration calls on the solver's stream."""
    import torch
    import torch.distributed as dist

    import paper_1501_07844_b200 as pf
    from paper_1501_07844_b200.dist import DistSolver

    dev = torch.device("cuda", local_rank)
    g, slab, D, kw = inputs_for_rank(cfg, rank, world)
    sha = inputs_sha256(D, kw) if rank == 0 else None
    ipc = args.transport == "ipc" and world > 1
    ds = DistSolver(_solver_factory(pf, cfg, g, D, kw, ipc), cfg.nz, rank, world, dev, transport=args.transport)
    del D
    s = ds.solver
    stream = torch.cuda.current_stream(dev)   # DistSolver puts the solver on this stream
    nzl = slab[1] - slab[0]
    labels = torch.empty((nzl, cfg.ny, cfg.nx), dtype=torch.uint8, device=dev)

    def step(evs=None):
        ds.reset()
        if evs is not None:
            evs[0].record(stream)
        ds.iterate(iters)
        if evs is not None:
            evs[1].record(stream)
        pf.pf_get_labeling(s.h, None, labels)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    kevs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = s.kernel_info()["kernel_launches"]
    clk = ClockSampler(local_rank) if clocks else None
    if clk:
        clk.__enter__()
        time.sleep(0.25)
    t_start.record(stream)
    for k in range(steps):
        step(kevs[k])
    t_end.record(stream)
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
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
    ds.close()
    V = cfg.nx * cfg.ny * nzl
    return {"ms": ms, "iter_ms": iter_ms, "info": info, "launches": int(launches), "V": V, "inputs_sha256": sha,
            "NF": info["flow_nodes"], "NL": len(g.leaves()), "slab": slab,
            "clocks": clk.summary() if clk else None}


def roofline(res, iters, steps, workload_name):
    info = res["info"]
    per_launch_ms = res["iter_ms"] / (iters * steps)
    alg = info["algorithmic_bytes_per_iteration"]
    achieved = alg / (per_launch_ms / 1e3) / 1e9
    peak, peak_src = _peaks()
    kernel = ("pf_iter_cluster" if info["cluster"] else "pf_iter_staged") if info["staged"] else "pf_iter_kernel"
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": _traffic(workload_name, kernel), "peak_source": peak_src, "kernel": kernel,
            "algorithmic_bytes_per_launch": alg, "mean_launch_ms": per_launch_ms, "src_hash": source_hash()}


def e2e_measure(cfg, rank, world, local_rank, args, iters, steps):
    """The same metric through the public API with HOST buffers: pf_create from pinned host D and S (H2D),
    the iterations, pf_get_labeling into pinned host u and argmax (D2H), pf_destroy -- wall clock, every
    step, max over ranks."""
    import torch
    import torch.distributed as dist

    import paper_1501_07844_b200 as pf
    from paper_1501_07844_b200.dist import DistSolver

    dev = torch.device("cuda", local_rank)
    g, slab, DH, kwH = inputs_for_rank(cfg, rank, world, pinned=True)
    nzl = slab[1] - slab[0]
    NL = len(DH)
    u_host = torch.empty((NL, nzl, cfg.ny, cfg.nx), dtype=torch.float32).pin_memory()
    lab_host = torch.empty((nzl, cfg.ny, cfg.nx), dtype=torch.uint8).pin_memory()
    h2d = sum(d.numel() * 4 for d in DH) + (kwH["s_shared"].numel() * 4 if "s_shared" in kwH else 0)
    d2h = u_host.numel() * 4 + lab_host.numel()
    ipc = args.transport == "ipc" and world > 1
    mk = _solver_factory(pf, cfg, g, DH, kwH, ipc)

    def one():
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

    one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    NF = cfg.graph().num_nodes - 1
    return {"value": cfg.nx * cfg.ny * cfg.nz * NF * iters * steps / float(te[0]) / 1e9, "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps,
            "path": f"pf_create(pinned host D,S) + pf_iterate({iters}) + pf_get_labeling(pinned host u, argmax) + "
                    "pf_destroy, wall clock"}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    cfg = workload(world, args.config)
    iters = args.iters or cfg.iters
    res = time_workload(cfg, rank, world, local_rank, args, iters, args.steps, args.warmup, clocks=True)
    vl_total = cfg.nx * cfg.ny * cfg.nz * res["NF"] * iters * args.steps
    value = vl_total / (res["ms"] / 1e3) / 1e9
    rl = roofline(res, iters, args.steps, cfg.name)
    # per-GPU denominator of C5's weak-scaling efficiency (N = 1 only)
    c5 = None
    if world == 1 and not args.no_c5slab and not args.config:
        c5cfg = c5slab_config()
        it5 = args.iters or c5cfg.iters
        st5 = max(1, min(args.steps, 3))
        r5 = time_workload(c5cfg, 0, 1, local_rank, args, it5, st5, max(3, min(args.warmup, 3)))
        c5 = {"workload": DESCR["C5slab"],
              "value": c5cfg.V * r5["NF"] * it5 * st5 / (r5["ms"] / 1e3) / 1e9, "unit": UNIT,
              "ms_per_iteration": r5["iter_ms"] / (it5 * st5), "steps": st5, "iterations_per_step": it5,
              "roofline": roofline(r5, it5, st5, "C5slab"),
              "kernel": {k: r5["info"][k] for k in ("tile_x", "tile_y", "z_chunk", "threads_per_cta", "ctas",
                                                    "regs_per_thread", "smem_bytes", "ctas_per_sm")}}
    e2e = None
    if not args.no_e2e:
        e2e = e2e_measure(cfg, rank, world, local_rank, args, iters, max(1, min(args.steps, 5 if world == 1 else 2)))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, dt, sample = cpu_oracle_rate(cfg, 2, _cpu_planes(cfg))
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample, "seconds": round(dt, 2)}
    if rank == 0:
        info = res["info"]
        exch = ""
        if world > 1:
            exch = (", halo exchange: " + ("fused CUDA-IPC peer stores" if args.transport == "ipc" else
                                           "NCCL P2P, overlapped" if dist.get_backend() == "nccl" else
                                           f"{dist.get_backend()} host-staged (validation only, not a measurement)"))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms"] / args.steps, "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": DESCR[cfg.name] + (f", z-sharded over {world} GPUs" if world > 1 else "") + exch,
                       "voxels": cfg.V, "voxels_per_gpu": res["V"], "flow_nodes": res["NF"],
                       "end_labels": res["NL"], "iterations_per_step": iters, "residual_check_every": 10,
                       "value_per_end_label": value * res["NL"] / res["NF"],
                       "inputs_sha256_rank0": res["inputs_sha256"],
                       "l2": "no flush: per-iteration state >> 126 MB L2 (C4 9.4 GB, C5 33-131 GB per GPU)",
                       "kernel": {k: info[k] for k in ("tile_x", "tile_y", "z_chunk", "threads_per_cta", "ctas",
                                                        "regs_per_thread", "smem_bytes", "ctas_per_sm")}},
            "roofline": rl,
            "c5slab": c5,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": res["launches"],
            "clocks": res["clocks"],
        }
        print(json.dumps(line), flush=True)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--iters", type=int, default=0, help="override iterations per step (default: the config's)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c5slab", action="store_true")
    ap.add_argument("--config", default="", choices=["", "C2", "C3", "C4", "C5", "C5slab", "C5small"],
                    help="experiments / code-path checks only: another workload than the contract's")
    ap.add_argument("--transport", choices=["nccl", "ipc"], default="nccl",
                    help="N > 1: halo exchange by NCCL P2P overlapped with the interior (default), or fused into "
                         "the kernels as CUDA-IPC peer stores (pf_ipc_*)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver launches it that way itself)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
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
