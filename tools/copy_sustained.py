"""Sustained device-copy bandwidth on this box, for context next to bench.py's roofline.

MEASURED_PEAKS.json's hbm_gbs is a burst figure (best of 10 single copies).  The bench kernel runs
back to back for ~1.3 s per 5 steps under sw_power_cap, so this measures the same copy (torch
copy_ of 1 Gi bf16 elements, read + write bytes) back to back for `seconds`, with the SM clock and
throttle reasons sampled as in bench.py.  It also times the pseudo-flow iteration (C2) in the same
process right after, so the two share one box and one thermal state.
usage: python tools/copy_sustained.py [seconds]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402


def copy_rate(seconds):
    n = 1 << 30
    a = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_()
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    evs = []
    t_end = time.time() + seconds
    with ClockSampler(0) as clk:
        while time.time() < t_end:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                b.copy_(a)
            e1.record()
            evs.append((e0, e1))
            e1.synchronize()
    ms = [x.elapsed_time(y) / 10 for x, y in evs]
    best = min(ms)
    tail = ms[len(ms) // 2:]   # second half: steady state under the power cap
    med = sorted(tail)[len(tail) // 2]
    by = 2 * n * 2
    return {"copy_gbs_burst": by / best / 1e6, "copy_gbs_sustained": by / med / 1e6, "batches": len(ms),
            "clocks": clk.summary()}


def pf_rate(seconds):
    import numpy as np
    import paper_1501_07844_b200 as pf
    import phantoms as P
    cfg = P.config("C2")
    inp = P.generate(cfg)
    g = inp.graph
    s = pf.Solver((cfg.nx, cfg.ny, cfg.nz), 3, (g.num_nodes, g.parent, g.child, g.weight),
                  [np.ascontiguousarray(inp.D[l]) for l in range(inp.D.shape[0])],
                  s_shared=np.ascontiguousarray(inp.s_field), c=cfg.c, tau=cfg.tau,
                  check_every=10)
    s.set_stream(torch.cuda.current_stream().cuda_stream)   # events below bracket the solver's launches
    s.iterate(30)
    torch.cuda.synchronize()
    info = s.kernel_info()
    ms = []
    t_end = time.time() + seconds
    with ClockSampler(0) as clk:
        while time.time() < t_end:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(torch.cuda.current_stream())
            s.iterate(100)
            e1.record(torch.cuda.current_stream())
            e1.synchronize()
            ms.append(e0.elapsed_time(e1) / 100)
    s.close()
    tail = ms[len(ms) // 2:]
    med = sorted(tail)[len(tail) // 2]
    by = info["algorithmic_bytes_per_iteration"]
    return {"pf_ms_per_iteration": med, "pf_gbs_sustained": by / med / 1e6, "clocks": clk.summary()}


if __name__ == "__main__":
    sec = float(sys.argv[1]) if len(sys.argv) > 1 else 6.0
    c = copy_rate(sec)
    p = pf_rate(sec)
    c2 = copy_rate(sec)
    out = {"copy_before": c, "pf_C2": p, "copy_after": c2,
           "pf_over_sustained_copy": p["pf_gbs_sustained"] / ((c["copy_gbs_sustained"] + c2["copy_gbs_sustained"]) / 2)}
    print(json.dumps(out), flush=True)
