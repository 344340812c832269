"""Small driver for ncu captures: builds one config's solver and runs a few iterations.
usage: python tools/prof_iter.py [C2|C3|C4|C5slab] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1501_07844_b200 as pf  # noqa: E402
import phantoms as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
if name == "C5slab":
    cfg = P.config("C5").resized(768, 768, 96, name="C5slab")
else:
    cfg = P.config(name)
inp = P.generate(cfg)
g = inp.graph
D = [np.ascontiguousarray(inp.D[l]) for l in range(inp.D.shape[0])]
kw = {"s_shared": inp.s_field} if inp.s_kind == "shared_field" else {"s_scalars": inp.s_scalars}
s = pf.Solver((cfg.nx, cfg.ny, cfg.nz), cfg.ndim, (g.num_nodes, g.parent, g.child, g.weight), D, c=cfg.c,
              tau=cfg.tau, check_every=10, **kw)
s.iterate(n, residual=True)
print(name, s.kernel_info())
if len(sys.argv) > 3:   # kernel info as JSON (tools/profile_round.sh: algorithmic bytes for the traffic entry)
    import json
    json.dump(s.kernel_info(), open(sys.argv[3], "w"))
s.close()
