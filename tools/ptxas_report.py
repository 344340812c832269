"""Registers / spills of every compiled kernel (from the ptxas -v logs of the last build).
usage: python tools/ptxas_report.py [substring]"""
import glob
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pat = sys.argv[1] if len(sys.argv) > 1 else "pf_iter_staged"
for f in sorted(glob.glob(os.path.join(ROOT, "paper_1501_07844_b200", "build_obj", "*.ptxas.txt"))):
    cur = None
    spill = ""
    for line in open(f):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            spill = f"spill st/ld {m.group(1)}/{m.group(2)}"
        m = re.search(r"Used (\d+) registers", line)
        if m and cur and pat in cur:
            t = re.search(r"ILi(-?\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)", cur)
            print(f"{'<' + ','.join(t.groups()) + '>' if t else cur:24s} regs {m.group(1):>4s}  {spill}")
            cur = None
