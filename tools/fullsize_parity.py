"""Full-size parity at the CONFIGURED iteration counts: the CUDA path through the C-ABI against the whole-volume
oracle (fp64, paper-exact, threaded over all host cores -- bit-identical to one thread, tests/test_oracle_pins.py).

usage (GPU box): python tools/fullsize_parity.py C2 C3 C4 C5small [--out profiles/r2/fullsize_parity.jsonl]
  C2, C3, C4, I2  BASELINE.json configs at full size and full iteration count (C3/C4 in both shifts with --both)
  C5small         the C5 fallback of SURVEY 8.4.5: 192^3, K = 16, same generator, 200 iterations, run as
                  8 z-slabs on one GPU (the 8-GPU decomposition, halos exchanged by pf_exchange_local)
One JSON line per case: max|du|, max|dq| (whole volume), argmax agreement, voxels above 1e-4, oracle time and
threads (the N-thread oracle timing next to bench.py's 1-thread cpu_baseline), GPU time of the same run.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import phantoms as P  # noqa: E402
from helpers import solver_from_inputs  # noqa: E402


def gpu_run(inp, n, shift, slabs):
    import torch
    import paper_1501_07844_b200 as pf
    t0 = time.perf_counter()
    if slabs > 1:
        solvers = [solver_from_inputs(inp, shift=shift, slab=b) for b in pf.solver.slab_bounds(inp.cfg.nz, slabs)]
        ss = pf.SlabSet(solvers, fused=all(s.kernel_info()["staged"] for s in solvers))
        ss.iterate(n)
        u, am = ss.labeling()
        q = ss.flows()
        ss.close()
    else:
        s = solver_from_inputs(inp, shift=shift)
        s.iterate(n)
        u, am = s.labeling()
        q = s.flows()
        s.close()
    torch.cuda.synchronize()
    return u, am, q, time.perf_counter() - t0


def case(name, shift, threads):
    if name == "C5small":
        cfg, slabs = P.config("C5").resized(192, 192, 192, name="C5small"), 8
    else:
        cfg, slabs = P.config(name), 1
    n = cfg.iters
    inp = P.generate(cfg)
    import hashlib
    h = hashlib.sha256(np.ascontiguousarray(inp.D).view(np.uint8))
    for f in inp.s_fields()[1:]:
        h.update(np.ascontiguousarray(f).view(np.uint8))
    u, am, q, gpu_s = gpu_run(inp, n, shift, slabs)
    O.set_threads(threads)
    t0 = time.perf_counter()
    ur, qr = O.run_inputs(inp, n, shift=shift)
    orc_s = time.perf_counter() - t0
    O.set_threads(1)
    du = np.abs(u - ur)
    big = int(np.count_nonzero(du.max(0) > 1e-4))
    du_max = float(du.max())
    del du
    dq_max = float(np.max(np.abs(q - qr)))
    agree = float(np.mean(am == O.argmax(ur)))
    vl = cfg.V * ur.shape[0] * n
    return {"case": f"{cfg.name} {cfg.nx}x{cfg.ny}x{cfg.nz}" + (f" as {slabs} z-slabs" if slabs > 1 else ""),
            "iterations": n, "shift": ["min", "none"][shift], "max_abs_du": du_max, "max_abs_dq": dq_max,
            "voxels_du_gt_1e-4": big, "argmax_agree": agree, "voxels": int(cfg.V),
            "pass": bool(du_max <= 1e-4 and dq_max <= 1e-4 and agree >= 0.9999),
            "oracle_s": round(orc_s, 1), "oracle_threads": threads,
            "oracle_gvl_it_s": round(vl / orc_s / 1e9, 4), "gpu_s_incl_create_and_copies": round(gpu_s, 2),
            "inputs_sha256": h.hexdigest()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="+")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2", "fullsize_parity.jsonl"))
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--both", action="store_true", help="also SHIFT_NONE (the literal listing)")
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    for name in a.cases:
        for shift in ([O.SHIFT_MIN, O.SHIFT_NONE] if a.both else [O.SHIFT_MIN]):
            r = case(name, shift, a.threads)
            print(json.dumps(r), flush=True)
            with open(a.out, "a") as fh:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
