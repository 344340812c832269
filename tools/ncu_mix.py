"""Executed-instruction mix by SASS opcode from an ncu report (--page source, sass).
usage: python tools/ncu_mix.py rep [n]"""
import collections
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
iE = h.index("Instructions Executed")
iS = h.index("Warp Stall Sampling (All Samples)")
mix = collections.Counter()
stall = collections.Counter()
for r in rows[2:]:
    ins = r[1].strip()
    if ins.startswith("@"):
        ins = ins.split(None, 1)[1]
    op = ins.split()[0] if ins else "?"
    mix[op] += float(r[iE] or 0)
    stall[op] += float(r[iS] or 0)
tot = sum(mix.values())
st = sum(stall.values())
print(f"total warp-instr {tot:.4g}")
for op, v in mix.most_common(n):
    print(f"{op:28s} {v / tot * 100:5.1f}%  stall {stall[op] / st * 100:5.1f}%")
