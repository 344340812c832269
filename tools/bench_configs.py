"""Measure every BASELINE.json config on one GPU (same method as bench.py) -> JSON lines.

usage: python tools/bench_configs.py [C1 C2 C3 C4 C5slab] [--steps K] [--oracle]
C5 (768^3, K=16) does not fit one GPU in the fused layout; "C5slab" is one rank's 768x768x96 z-slab
of it (the weak-scaling unit of the 8-GPU run).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1501_07844_b200 as pf  # noqa: E402
import phantoms as P  # noqa: E402


def cfg_of(name):
    if name == "C5slab":
        return P.config("C5").resized(768, 768, 96, name="C5slab")
    if name in ("W8", "W8s", "W16s"):   # diagnostics, C5's recipe: K = 8 (one-CTA staged kernel) on 768^2 / 256^2
        # planes, K = 16 (cluster kernel) on 256^2 planes -- the same voxel count as C5slab
        K = 16 if name == "W16s" else 8
        nx, nz = (768, 96) if name == "W8" else (256, 864)
        return P.Config(name, 3, nx, nx, nz, "potts", K, 60 if K == 16 else 28, 0.15, "abs", "edge", 0.05, 200,
                        seed=1005)
    if name in ("T2", "T3", "T4"):   # f3 demonstration volumes: C2's recipe (256^3, edge S) with K = 2..4 labels
        K = int(name[1])
        return P.Config(name, 3, 256, 256, 256, "potts", K, 4 * K, 0.15, "sq", "edge", 0.05, 300, seed=2020)
    return P.config(name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C1", "C2", "C3", "C4", "C5slab", "I2"])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--d-bf16", action="store_true", help="store D as bf16 (pf_config.d_bf16)")
    ap.add_argument("--alm", action="store_true", help="explicit-flow ALM comparison arm (Potts configs)")
    ap.add_argument("--u-half", action="store_true", help="lambda = log2 u stored as binary16 (pf_config.u_half)")
    ap.add_argument("--linf", action="store_true", help="anisotropic capacities: the l-inf box (dual of l1-TV)")
    ap.add_argument("--tblock", type=int, default=0, help="2: two iterations per HBM pass (pf_config.tblock)")
    args = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    dev = torch.device("cuda", 0)
    for name in args.configs:
        cfg = cfg_of(name)
        inp = P.generate(cfg)
        g = inp.graph
        D = [torch.from_numpy(np.ascontiguousarray(inp.D[l])).to(dev) for l in range(inp.D.shape[0])]
        if cfg.kind == "ishikawa":
            fac = np.zeros(g.num_nodes, np.float32)
            fac[1:len(D)] = 1.0
            kw = {"s_scaled": (fac, torch.from_numpy(inp.s_field).to(dev))}
        elif inp.s_kind == "shared_field":
            kw = {"s_shared": torch.from_numpy(inp.s_field).to(dev)}
        else:
            kw = {"s_scalars": inp.s_scalars}
        extra = {"d_bf16": args.d_bf16, "u_half": args.u_half, "cap": pf.PF_CAP_LINF if args.linf else pf.PF_CAP_L2,
                 "tblock": args.tblock}
        c, tau = cfg.c, cfg.tau
        if args.alm:
            extra["method"] = pf.PF_METHOD_EXPLICIT_ALM
            c, tau = 0.3, 0.11   # oracle/alm.py potts_alm defaults
        s = pf.Solver((cfg.nx, cfg.ny, cfg.nz), cfg.ndim, (g.num_nodes, g.parent, g.child, g.weight), D, c=c,
                      tau=tau, check_every=10, **extra, **kw)
        stream = torch.cuda.current_stream(dev)
        s.set_stream(stream.cuda_stream)
        labels = torch.empty((cfg.nz, cfg.ny, cfg.nx), dtype=torch.uint8, device=dev)
        n = cfg.iters

        def step(ev=None):
            s.reset()
            if ev:
                ev[0].record(stream)
            s.iterate(n)
            if ev:
                ev[1].record(stream)
            pf.pf_get_labeling(s.h, None, labels)

        step()
        torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(args.steps):
            step(evs[k])
        t1.record(stream)
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1) / args.steps
        it_ms = sum(a.elapsed_time(b) for a, b in evs) / (args.steps * n)
        info = s.kernel_info()
        NL = len(D)
        V = cfg.V
        r = s.iterate(0, True)
        e, f = s.energy()
        s.close()
        line = {"config": name, "method": "explicit-flow ALM" if args.alm else "pseudo-flow",
                "d_dtype": "bf16" if args.d_bf16 else "f32", "u_storage": "binary16 lambda" if args.u_half else "f32 lambda",
                "capacity": "linf" if args.linf else "l2", "tblock": info["tblock"],
                "dims": [cfg.nx, cfg.ny, cfg.nz], "end_labels": NL, "nodes": g.num_nodes - 1,
                "iterations": n, "ms_per_solve": ms, "ms_per_iteration": it_ms,
                "gvl_it_per_s": V * NL * n / (ms / 1e3) / 1e9,
                "gvnode_it_per_s": V * (g.num_nodes - 1) * n / (ms / 1e3) / 1e9,
                "algorithmic_bytes_per_iteration": info["algorithmic_bytes_per_iteration"],
                "achieved_gbs": info["algorithmic_bytes_per_iteration"] / (it_ms / 1e3) / 1e9,
                "frac_of_measured_peak": info["algorithmic_bytes_per_iteration"] / (it_ms / 1e3) / 1e9 / peak,
                "kernel": {k: info[k] for k in ("staged", "tile_y", "z_chunk", "ctas", "regs_per_thread",
                                                "smem_bytes", "work_items")},
                "device_bytes": info["device_bytes"], "final_primal": e, "final_dual": f}
        if args.oracle:
            import oracle as O
            planes = max(1, min(cfg.nz, int(4e6 // (cfg.nx * cfg.ny))))
            sub = P.generate(cfg, (0, planes, 0, cfg.ny, 0, cfg.nx))
            t = time.perf_counter()
            O.run_inputs(sub, 2)
            dt = time.perf_counter() - t
            rate = sub.D.size * 2 / dt
            line["oracle_1thread_gvl_it_per_s"] = rate / 1e9
            line["oracle_1thread_full_run_s_extrapolated"] = V * NL * n / rate
        print(json.dumps(line), flush=True)
        del D, kw, labels
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
