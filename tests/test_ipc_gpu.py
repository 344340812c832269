"""Fused halo exchange across processes (transport="ipc"): ranks on ONE GPU here, each a separate process
with its own slab solver; the iteration kernels store their boundary planes straight into the neighbours'
CUDA-IPC-mapped halo planes, ordered by interprocess events (no kernel waits on another rank's kernel:
the ordering is stream-event based).  The decomposed run must equal the single-domain run bit for bit."""
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, name, dims, iters, outdir):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import phantoms as P
    from paper_1501_07844_b200.dist import DistSolver

    inp = P.generate(P.config(name).resized(*dims))

    def make(slab):
        return _ipc_solver(inp, slab)

    ds = DistSolver(make, inp.cfg.nz, rank, world, torch.device("cuda", 0), transport="ipc")
    ds.iterate(iters // 2 + 3)
    ds.reset()                                   # re-init protocol: the run below starts from scratch
    r = ds.iterate(iters, residual=True)
    u, a = ds.solver.labeling()
    q = ds.solver.flows()
    e = ds.energy()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), u=u, a=a, q=q, r=np.float64(r), e=np.array(e))
    dist.barrier()
    ds.close()
    dist.destroy_process_group()


def _ipc_solver(inp, slab):
    import paper_1501_07844_b200 as pf
    from helpers import CAP
    cfg, g = inp.cfg, inp.graph
    z0, z1 = slab
    zt = min(z1 + 1, cfg.nz)
    D = [np.ascontiguousarray(inp.D[l, z0:zt]) for l in range(inp.D.shape[0])]
    kw = ({"s_shared": np.ascontiguousarray(inp.s_field[z0:z1])} if inp.s_kind == "shared_field"
          else {"s_scalars": inp.s_scalars})
    return pf.Solver((cfg.nx, cfg.ny, cfg.nz), cfg.ndim, (g.num_nodes, g.parent, g.child, g.weight), D, c=cfg.c,
                     tau=cfg.tau, cap=CAP[cfg.cap], check_every=10, slab=(z0, z1), ipc=True, **kw)


@pytest.mark.parametrize("name,dims,world,iters", [("C2", (40, 33, 24), 2, 30), ("C5", (36, 21, 17), 3, 21),
                                                   ("C4", (33, 30, 14), 2, 20)])
def test_ipc_fused_exchange_bitwise(name, dims, world, iters):
    import torch.multiprocessing as mp

    import phantoms as P
    from helpers import solver_from_inputs

    inp = P.generate(P.config(name).resized(*dims))
    ref = solver_from_inputs(inp)
    if not ref.kernel_info()["staged"]:
        pytest.skip("fused halo stores need the TMA-staged kernels")
    r_ref = ref.iterate(iters, residual=True)
    u_ref, a_ref = ref.labeling()
    q_ref = ref.flows()
    e_ref = ref.energy()
    ref.close()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank, args=(world, _free_port(), name, dims, iters, d), nprocs=world, join=True)
        parts = [np.load(os.path.join(d, f"r{r}.npz")) for r in range(world)]
        u = np.concatenate([p["u"] for p in parts], axis=1)
        a = np.concatenate([p["a"] for p in parts], axis=0)
        q = np.concatenate([p["q"] for p in parts], axis=2)
        assert np.array_equal(u, u_ref) and np.array_equal(a, a_ref) and np.array_equal(q, q_ref)
        assert all(float(p["r"]) == r_ref for p in parts)          # residual: max over ranks
        e = parts[0]["e"]
        assert abs(e[0] - e_ref[0]) <= 1e-9 * abs(e_ref[0]) and abs(e[1] - e_ref[1]) <= 1e-9 * abs(e_ref[0])


def test_ipc_protocol_errors():
    import paper_1501_07844_b200 as pf
    import phantoms as P
    from helpers import solver_from_inputs

    inp = P.generate(P.config("C2").resized(40, 17, 12))
    s = solver_from_inputs(inp, slab=(0, 6))            # not created with ipc=True
    with pytest.raises(pf.PFError) as ei:
        pf.pf_ipc_export(s.h)
    assert ei.value.status == pf.PF_ERR_STATE
    with pytest.raises(pf.PFError) as ei:
        pf.pf_ipc_step(s.h)
    assert ei.value.status == pf.PF_ERR_STATE
    s.close()
    a, b = _ipc_solver(inp, (0, 6)), _ipc_solver(inp, (6, 12))
    if not a.kernel_info()["staged"]:
        pytest.skip("fused halo stores need the TMA-staged kernels")
    blob_a = pf.pf_ipc_export(a.h)
    with pytest.raises(pf.PFError) as ei:               # a's own blob is not the slab above it
        pf.pf_ipc_link(a.h, None, blob_a)
    assert ei.value.status == pf.PF_ERR_INVALID
    a.close()
    b.close()
