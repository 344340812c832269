"""Replace a workload's entry in profiles/ncu_traffic.json by the per-launch DRAM bytes of an ncu app-range
capture (tools/prof_range.py: N back-to-back iterations in one range) -- for kernels whose single-launch kernel
replay is not representative (the cluster kernel).
usage: python tools/traffic_from_range.py <range.csv> <workload> <iterations> [traffic.json]"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path, workload, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
tj_path = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "profiles", "ncu_traffic.json")
rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
h = rows[0]
v = {r[h.index("Metric Name")]: float(r[h.index("Metric Value")]) for r in rows[1:]}
per_launch = (v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]) / n
tj = json.load(open(tj_path))
for e in tj["entries"]:
    if e["workload"] == workload:
        e["single_launch_kernel_replay"] = {k: e[k] for k in ("dram_bytes_per_launch", "traffic_over_algorithmic",
                                                               "gpu__time_duration") if k in e}
        e["dram_bytes_per_launch"] = per_launch
        e["traffic_over_algorithmic"] = per_launch / e["algorithmic_bytes_per_launch"]
        e["method"] = f"ncu --replay-mode app-range over {n} back-to-back iterations / {n} ({os.path.basename(path)})"
        e["dram_bytes_read_per_launch"] = v["dram__bytes_read.sum"] / n
        e["dram_bytes_write_per_launch"] = v["dram__bytes_write.sum"] / n
        e.pop("gpu__time_duration", None)
        print(json.dumps(e, indent=1))
json.dump(tj, open(tj_path, "w"), indent=1)
