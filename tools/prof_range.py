"""Sustained-sequence profile: N back-to-back iterations inside one cudaProfilerStart/Stop range, for
ncu --replay-mode app-range (total DRAM bytes of the whole sequence, no per-kernel serialisation).
usage: ncu --replay-mode app-range --profile-from-start off --metrics ... python tools/prof_range.py C5slab 20 [warm-up iterations]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1501_07844_b200 as pf  # noqa: E402
import phantoms as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 30   # iterations before the profiled range
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bench_configs import cfg_of  # noqa: E402

cfg = cfg_of(name)
inp = P.generate(cfg)
g = inp.graph
D = [np.ascontiguousarray(inp.D[l]) for l in range(inp.D.shape[0])]
kw = {"s_shared": inp.s_field} if inp.s_kind == "shared_field" else {"s_scalars": inp.s_scalars}
s = pf.Solver((cfg.nx, cfg.ny, cfg.nz), cfg.ndim, (g.num_nodes, g.parent, g.child, g.weight), D, c=cfg.c,
              tau=cfg.tau, check_every=10, **kw)
s.iterate(warm)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
s.iterate(n)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
info = s.kernel_info()
print(name, "iterations", n, "algorithmic bytes per iteration", info["algorithmic_bytes_per_iteration"])
s.close()
