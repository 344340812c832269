"""Diagnostic: is the iteration's result at N iterations determined to 1e-4 by its inputs at all?  Runs the fp64
oracle twice -- on D and on D (1 + delta) with delta = 1e-12 (far below fp32's 6e-8 resolution) -- and reports
how far the two fp64 trajectories separate.  A separation >> 1e-4 means the listing is ill-conditioned there:
no implementation in any precision below "exact" can be held to 1e-4 against an fp64 run.
usage: PYTHONPATH=. python tools/conditioning.py C3 64 64 64 300 1 [...]   (name nx ny nz iters shift)"""
import os
import sys

import numpy as np

import oracle as O
import phantoms as P

O.set_threads(os.cpu_count() or 1)
DELTA = float(os.environ.get("DELTA", "1e-12"))
args = sys.argv[1:] or ["C3", "64", "64", "64", "300", "1"]
for i in range(0, len(args), 6):
    name, nx, ny, nz, n, shift = args[i:i + 6]
    inp = P.generate(P.config(name).resized(int(nx), int(ny), int(nz)))
    ua, qa = O.run_inputs(inp, int(n), shift=int(shift))
    inp.D = (inp.D.astype(np.float64) * (1 + DELTA))
    ub, qb = O.run_inputs(inp, int(n), shift=int(shift))
    du = np.abs(ua - ub)
    print(f"{name} {nx}x{ny}x{nz} n={n} shift={'none' if int(shift) else 'min'}: fp64 vs fp64 with D(1+{DELTA:g}): "
          f"max|du| {du.max():.3g} max|dq| {np.abs(qa - qb).max():.3g} voxels du>1e-4 {int((du.max(0) > 1e-4).sum())}"
          f"/{du[0].size} argmax {np.mean(np.argmax(ua, 0) == np.argmax(ub, 0)) * 100:.4f}%", flush=True)
