"""DistSolver's process-group transport (the path bench.py uses over NCCL) exercised with 2-3 processes on
ONE GPU over gloo: the halo exchange is host-mediated, so no rank's kernel waits on another's.  The
decomposed run (and its resume from per-rank checkpoints) must equal the single-domain run bitwise.  usage: python tools/dist_one_gpu.py [world]"""
import os
import socket
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import phantoms as P
    from helpers import solver_from_inputs
    from paper_1501_07844_b200.dist import DistSolver
    cfg = P.config("C2").resized(40, 33, 24)
    inp = P.generate(cfg)
    ds = DistSolver(lambda slab: solver_from_inputs(inp, slab=slab), cfg.nz, rank, world, torch.device("cuda", 0))
    r = ds.iterate(20, residual=True)
    torch.cuda.synchronize()
    u, _ = ds.solver.labeling()
    # checkpoint / resume through DistSolver (rank files + halo refresh), then 7 more iterations
    prefix = os.path.join(os.environ.get("CK_DIR", "/tmp"), "dist_ck")
    ds.save(prefix)
    ds2 = DistSolver(lambda slab: solver_from_inputs(inp, slab=slab), cfg.nz, rank, world, torch.device("cuda", 0))
    ds2.iterate(3)
    ds2.load(prefix)
    ds2.iterate(7)
    torch.cuda.synchronize()
    u2, _ = ds2.solver.labeling()
    out[rank] = (ds.slab, u, ds.solver.flows(), r, u2, ds2.solver.flows())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = mp.Manager().dict()
    mp.spawn(worker, args=(world, port, out), nprocs=world, join=True)
    import phantoms as P
    from helpers import solver_from_inputs
    cfg = P.config("C2").resized(40, 33, 24)
    ref = solver_from_inputs(P.generate(cfg))
    r_ref = ref.iterate(20, residual=True)
    u_ref, _ = ref.labeling()
    q_ref = ref.flows()
    ref.iterate(7)
    u_ref2, _ = ref.labeling()
    q_ref2 = ref.flows()
    ok = True
    for rank in range(world):
        (z0, z1), u, q, r, u2, q2 = out[rank]
        ok &= np.array_equal(u, u_ref[:, z0:z1]) and np.array_equal(q, q_ref[:, :, z0:z1])
        ok &= r == r_ref
        ok &= np.array_equal(u2, u_ref2[:, z0:z1]) and np.array_equal(q2, q_ref2[:, :, z0:z1])
    print("dist_one_gpu", world, "bitwise" if ok else "MISMATCH", flush=True)
    sys.exit(0 if ok else 1)
