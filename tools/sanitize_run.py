"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
python tools/sanitize_run.py   (run under: compute-sanitizer --tool <tool> python tools/sanitize_run.py)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import dataclasses  # noqa: E402

import phantoms as P  # noqa: E402
from helpers import solver_from_inputs  # noqa: E402

import paper_1501_07844_b200 as pf  # noqa: E402

cases = [("C2", (40, 17, 9), {}), ("C4", (33, 18, 7), {}), ("C5", (41, 10, 6), {}), ("I2", (35, 9, 5), {}),
         ("C2", (37, 12, 6), {"d_bf16": True}), ("C2", (36, 12, 5), {"method": pf.PF_METHOD_EXPLICIT_ALM}),
         ("C3", (30, 12, 5), {"method": pf.PF_METHOD_EXPLICIT_ALM})]
for name, dims, kw in cases:
    inp = P.generate(P.config(name).resized(*dims))
    s = solver_from_inputs(inp, **kw)
    s.iterate(12, residual=True)
    s.labeling()
    s.energy()
    s.close()
    print("ok", name, dims, kw, flush=True)
# slabs: fused linked kernels and the split schedule
for fused in (True, False):
    inp = P.generate(P.config("C5").resized(36, 9, 8))
    ss = pf.SlabSet([solver_from_inputs(inp, slab=b) for b in pf.solver.slab_bounds(8, 2)], phased=not fused,
                    fused=fused)
    ss.iterate(5)
    ss.close()
    print("ok slabs fused" if fused else "ok slabs phased", flush=True)
