"""GPU parity of the generic path (pf_generic.cu): label DAGs beyond the compiled kernel set (> 4 internal or
> 16 non-source nodes), up to SURVEY 8.6's limits of 31 non-source nodes and 16 end labels, vs the CPU oracle
(Alg. 2) on the same seeded inputs -- bar as north_star: max|du|, max|dq| <= 1e-4, argmax >= 99.99 %.
Plus: the generic kernels forced on a compiled-set graph are bitwise the dense compiled kernels (same arithmetic)."""
import dataclasses

import numpy as np
import pytest

import oracle as O
import phantoms as P
from helpers import compare, solver_from_inputs

pytestmark = pytest.mark.gpu


def wide_inputs(ni, nl, dims, seed, s_kind="per_node_uniform", cap="l2"):
    base = P.config("C3")
    cfg = dataclasses.replace(base, name=f"W{ni}x{nl}", kind="wide", wide_ni=ni, classes=nl, seed=seed,
                              nx=dims[0], ny=dims[1], nz=dims[2], s_kind=s_kind, s_value=0.05, cap=cap,
                              n_shapes=3 * nl)
    return P.generate(cfg)


@pytest.mark.parametrize("ni,nl,dims,n,s_kind,cap", [
    (5, 6, (40, 36, 12), 300, "per_node_uniform", "l2"),    # 11 nodes, > 4 internal
    (8, 12, (40, 20, 10), 200, "edge", "l2"),                # 20 nodes, shared edge-weighted S field
    (15, 16, (33, 17, 9), 200, "per_node_uniform", "linf"),  # 31 nodes, 16 end labels: the SURVEY 8.6 maximum
    (2, 16, (36, 9, 5), 150, "per_node_uniform", "l2"),      # 18 nodes, few internal
])
def test_generic_graph_parity(ni, nl, dims, n, s_kind, cap):
    inp = wide_inputs(ni, nl, dims, seed=100 + ni, s_kind=s_kind, cap=cap)
    assert len(inp.graph.leaves()) == nl and inp.graph.num_nodes == ni + nl + 1
    s = solver_from_inputs(inp)
    l0 = s.kernel_info()["kernel_launches"]
    s.iterate(n)
    launches = s.kernel_info()["kernel_launches"] - l0
    u, am = s.labeling()
    q = s.flows()
    s.close()
    assert launches == 2 * n   # two passes per iteration (masses, flows)
    ur, qr = O.run_inputs(inp, n)
    compare(u, q, ur, qr)
    assert np.array_equal(am, O.argmax(u))


def test_generic_energies_and_node_labeling():
    """The energy kernel and the intermediate labelings on a 31-node graph vs the oracle's."""
    from oracle import energy as E
    inp = wide_inputs(15, 16, (24, 20, 10), seed=7)
    g = inp.graph
    s = solver_from_inputs(inp)
    s.iterate(60)
    e, f = s.energy()
    ur, qr = O.run_inputs(inp, 60)
    S = np.zeros((g.num_nodes,) + inp.shape)
    for v in range(1, g.num_nodes):
        S[v] = inp.s_fields()[v]
    eo = E.primal(ur, inp.D.astype(np.float64), S, g.num_nodes, g.parent, g.child, g.weight, inp.cfg.ndim)
    fo = E.dual(qr, inp.D.astype(np.float64), g.num_nodes, g.parent, g.child, g.weight, inp.cfg.ndim)
    assert e >= f - 1e-9 * abs(e)
    assert abs(e - eo) <= 1e-4 * abs(eo) and abs(f - fo) <= 1e-4 * abs(eo)
    # u of internal node 1 = sum over end labels of W_(1, L) u_L: W from the oracle's graph walk
    W = np.zeros(len(g.leaves()))
    leaves = g.leaves()
    def walk(v, w):
        if v in leaves:
            W[leaves.index(v)] += w
        for p, c, wt in g.edges:
            if p == v:
                walk(c, w * wt)
    walk(1, 1.0)
    un = s.node_labeling(1)
    s.close()
    assert np.max(np.abs(un - np.tensordot(W, ur, axes=1))) <= 1e-4


@pytest.mark.parametrize("name,dims", [("C4", (40, 36, 20)), ("C3", (33, 17, 9)), ("C2", (40, 20, 12))])
def test_generic_bitwise_equals_dense_compiled(name, dims, monkeypatch):
    """PF_GENERIC=1 puts a compiled-set graph on the generic kernels: same operations in the same order as the
    dense-weight compiled kernel (PF_DENSE_GRAPH=1), so u and q are bitwise equal."""
    inp = P.generate(P.config(name).resized(*dims))
    out = []
    for generic in ("0", "1"):
        monkeypatch.setenv("PF_GENERIC", generic)
        monkeypatch.setenv("PF_DENSE_GRAPH", "1")
        s = solver_from_inputs(inp)
        s.iterate(40)
        u, _ = s.labeling()
        out.append((u, s.flows(), s.kernel_info()["staged"]))
        s.close()
    assert out[0][2] == 1 and out[1][2] == 0
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


def test_generic_limits():
    import paper_1501_07844_b200 as pf
    g = P.wide_dag(16, 16, 3)   # 32 non-source nodes: beyond SURVEY 8.6
    D = [np.zeros((4, 8, 8), np.float32) for _ in range(16)]
    with pytest.raises(pf.PFError) as ei:
        pf.Solver((8, 8, 4), 3, (g.num_nodes, g.parent, g.child, g.weight), D,
                  s_scalars=np.full(g.num_nodes, 0.1, np.float32))
    assert ei.value.status == pf.PF_ERR_UNSUPPORTED
    g = P.wide_dag(8, 12, 2)    # generic graphs: whole volumes only
    D = [np.zeros((3, 8, 8), np.float32) for _ in range(12)]   # the slab's planes + the plane above
    with pytest.raises(pf.PFError) as ei:
        pf.Solver((8, 8, 4), 3, (g.num_nodes, g.parent, g.child, g.weight), D,
                  s_scalars=np.full(g.num_nodes, 0.1, np.float32), slab=(0, 2))
    assert ei.value.status == pf.PF_ERR_UNSUPPORTED
