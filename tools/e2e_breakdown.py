"""Where the end-to-end step of bench.py spends its time (pf_create / iterate / labeling / destroy)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench as B  # noqa: E402
import paper_1501_07844_b200 as pf  # noqa: E402

base, cfg = B._workload(1)
g, slab, D, S = B._inputs_for_rank(cfg, 0, 1, pinned=True)
NL = len(D)
u_host = torch.empty((NL, cfg.nz, cfg.ny, cfg.nx), dtype=torch.float32).pin_memory()
lab = torch.empty((cfg.nz, cfg.ny, cfg.nx), dtype=torch.uint8).pin_memory()
hot = None
if "--hot" in sys.argv:   # as in bench.py: the benchmark solver stays alive and the GPU is hot
    hot = pf.Solver((cfg.nx, cfg.ny, cfg.nz), 3, (g.num_nodes, g.parent, g.child, g.weight), D, s_shared=S,
                    c=cfg.c, tau=cfg.tau, check_every=10)
    for _ in range(8):
        hot.reset()
        hot.iterate(300)
    torch.cuda.synchronize()
for rep in range(4):
    t = [time.perf_counter()]
    s = pf.Solver((cfg.nx, cfg.ny, cfg.nz), 3, (g.num_nodes, g.parent, g.child, g.weight), D, s_shared=S,
                  c=cfg.c, tau=cfg.tau, check_every=10)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    s.iterate(300)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    s.labeling(u_host, lab)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    s.close()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = [round((b - a) * 1e3, 1) for a, b in zip(t, t[1:])]
    print("create / iterate(300) / labeling / destroy ms:", d, flush=True)
