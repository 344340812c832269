"""ncu driver for the explicit-flow ALM arm: python tools/prof_alm.py C3 [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1501_07844_b200 as pf  # noqa: E402
import phantoms as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = P.config(name)
inp = P.generate(cfg)
g = inp.graph
D = [np.ascontiguousarray(inp.D[l]) for l in range(inp.D.shape[0])]
kw = {"s_shared": inp.s_field} if inp.s_kind == "shared_field" else {"s_scalars": inp.s_scalars}
s = pf.Solver((cfg.nx, cfg.ny, cfg.nz), cfg.ndim, (g.num_nodes, g.parent, g.child, g.weight), D, c=0.3,
              tau=0.05 if cfg.kind != "potts" else 0.11, check_every=10, method=pf.PF_METHOD_EXPLICIT_ALM, **kw)
s.iterate(n)
s.close()
