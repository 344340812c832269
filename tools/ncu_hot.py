"""Top stall sites (SASS) of an ncu report with --import-source.  usage: python tools/ncu_hot.py rep [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
d = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
tot = sum(float(r[iS] or 0) for r in d)
print("total samples", tot, "warp-instr", sum(float(r[iE] or 0) for r in d))
for r in sorted(d, key=lambda r: -float(r[iS] or 0))[:n]:
    print(f"{float(r[iS]) / tot * 100:5.1f}% {r[iE]:>10s} {r[0][-5:]} {r[1][:100]}")
