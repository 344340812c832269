"""ncu driver: one T-volume (C2 recipe, K labels, 256^3) solver, a few iterations, tblock as given.
usage: python tools/prof_tb.py T4 2 [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import numpy as np  # noqa: E402

import paper_1501_07844_b200 as pf  # noqa: E402
from bench_configs import cfg_of  # noqa: E402
import phantoms as P  # noqa: E402

name, tb = sys.argv[1], int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 6
cfg = cfg_of(name)
inp = P.generate(cfg)
g = inp.graph
D = [np.ascontiguousarray(inp.D[l]) for l in range(inp.D.shape[0])]
s = pf.Solver((cfg.nx, cfg.ny, cfg.nz), 3, (g.num_nodes, g.parent, g.child, g.weight), D, c=cfg.c, tau=cfg.tau,
              check_every=10, s_shared=inp.s_field, tblock=tb)
s.iterate(n, residual=True)
print(name, tb, s.kernel_info())
s.close()
