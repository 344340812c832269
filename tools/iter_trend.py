"""Launch time of the fused iteration as a function of the iteration index (host clock around synchronised blocks
of iterations): does the kernel slow down as the flows saturate / the CTAs drift apart?
usage: [PF_LIB=...] python tools/iter_trend.py C5slab [iterations] [block]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1501_07844_b200 as pf  # noqa: E402
import phantoms as P  # noqa: E402
from bench_configs import cfg_of  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5slab"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
blk = int(sys.argv[3]) if len(sys.argv) > 3 else 10
cfg = cfg_of(name)
inp = P.generate(cfg)
g = inp.graph
D = [np.ascontiguousarray(inp.D[l]) for l in range(inp.D.shape[0])]
kw = {"s_shared": inp.s_field} if inp.s_kind == "shared_field" else {"s_scalars": inp.s_scalars}
s = pf.Solver((cfg.nx, cfg.ny, cfg.nz), cfg.ndim, (g.num_nodes, g.parent, g.child, g.weight), D, c=cfg.c,
              tau=cfg.tau, check_every=10, **kw)
for rep in range(2):   # second pass after pf_reset: same state sequence, warmed-up clocks
    s.reset()
    torch.cuda.synchronize()
    ms = []
    for i in range(n // blk):   # the solver runs on its own stream: host clock around a synchronised block
        t0 = time.perf_counter()
        s.iterate(blk)
        torch.cuda.synchronize()
        ms.append((time.perf_counter() - t0) * 1e3 / blk)
    print(name, os.environ.get("PF_LIB", "libpf.so"), os.environ.get("PF_STRIP", ""), "pass", rep,
          "ms/iteration per block of", blk, ":", " ".join(f"{m:.3f}" for m in ms), flush=True)
s.close()
