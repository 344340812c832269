"""Repeat a configuration many times and check the result is bitwise stable (races in the cluster
exchange would show up as a differing or failing run).  usage: python tools/stress_cluster.py C5slab 20 30"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import phantoms as P  # noqa: E402
from helpers import solver_from_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5slab"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cfg = P.config("C5").resized(768, 768, 96, name="C5slab") if name == "C5slab" else P.config(name)
inp = P.generate(cfg)
s = solver_from_inputs(inp)
ref = None
bad = 0
for r in range(reps):
    s.reset()
    s.iterate(iters)
    u, _ = s.labeling()
    h = (float(np.sum(u, dtype=np.float64)), u[:, ::7, ::5, ::3].tobytes())
    if ref is None:
        ref = h
    elif h != ref:
        bad += 1
        print("run", r, "differs", h[0], ref[0], flush=True)
print(name, "reps", reps, "iters", iters, "differing runs", bad, s.kernel_info()["staged"], flush=True)
