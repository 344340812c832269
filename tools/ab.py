"""A/B timing of library builds in ONE GPU session (boxes differ from call to call, so only
interleaved runs on the same GPU compare kernel variants).
usage: python tools/ab.py --libs libpf_ref.so libpf.so libpf.so:PF_CLUSTER=0 --configs C2 C5slab [--rounds 3] [--alm]
Each (round, config, lib) runs tools/bench_configs.py in a fresh process with PF_LIB=<lib>."""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--libs", nargs="+", required=True)
ap.add_argument("--configs", nargs="+", default=["C2", "C5slab"])
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--alm", action="store_true", help="time the explicit-flow ALM arm (bench_configs.py --alm)")
ap.add_argument("--extra", default="", help="extra bench_configs.py arguments, e.g. '--tblock 2'")
args = ap.parse_args()
res = {}
for r in range(args.rounds):
    for c in args.configs:
        for lib in args.libs:
            # "libname.so[:VAR=value,...]": extra environment for that arm (e.g. PF_CLUSTER=0)
            name, _, extra = lib.partition(":")
            env = dict(os.environ, PF_LIB=name)
            for kv in filter(None, extra.split(",")):
                k, _, v = kv.partition("=")
                env[k] = v
            pr = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bench_configs.py"), c, "--steps",
                                 str(args.steps)] + (["--alm"] if args.alm else []) + args.extra.split(), env=env, capture_output=True,
                                text=True)
            out = pr.stdout
            if pr.returncode != 0:
                print(json.dumps({"round": r, "config": c, "lib": lib, "failed": pr.returncode,
                                  "stderr": pr.stderr[-600:]}), flush=True)
            for line in out.splitlines():
                try:
                    d = json.loads(line)
                except ValueError:
                    continue
                res.setdefault((c, lib), []).append(d["ms_per_iteration"])
                print(json.dumps({"round": r, "config": c, "lib": lib, "ms_per_iteration": d["ms_per_iteration"],
                                  "frac": d["frac_of_measured_peak"], "regs": d["kernel"]["regs_per_thread"]}),
                      flush=True)
for (c, lib), v in sorted(res.items()):
    print(f"{c:8s} {lib:20s} median {statistics.median(v):.4f} ms/it  all {[round(x, 4) for x in v]}")
