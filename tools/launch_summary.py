"""Per-kernel share of a step from an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python tools/launch_summary.py launches.csv out.json "<command>" """
import csv
import json
import re
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
iN, iV = h.index("Kernel Name"), h.index("Metric Value")
agg = {}
for r in rows[1:]:
    name = re.sub(r"\(.*", "", r[iN]).strip()
    name = re.sub(r"^void ", "", name)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(r[iV])
tot = sum(v[1] for v in agg.values())
out = {"command": sys.argv[3] if len(sys.argv) > 3 else "", "kernels": {
    k: {"launches": n, "total_ns": t, "mean_ns": t / n, "share": t / tot} for k, (n, t) in agg.items()}}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
