"""CPU: the seeded wide label DAGs the generic-path GPU tests use (phantoms.wide_dag) are valid Alg. 2 inputs --
acyclic, the requested end-label count, W_(S,L) = 1 for every end label (reading R9) -- and the
oracle keeps sum_L u_L = 1 on them."""
import dataclasses

import numpy as np
import pytest

import oracle as O
import phantoms as P


@pytest.mark.parametrize("ni,nl,seed", [(5, 6, 105), (8, 12, 108), (15, 16, 115), (2, 16, 102), (15, 16, 3)])
def test_wide_dag_valid(ni, nl, seed):
    g = P.wide_dag(ni, nl, seed)
    assert g.num_nodes == ni + nl + 1 and len(g.leaves()) == nl
    assert O.topo_order(g.num_nodes, g.parent, g.child, g.weight) is not None
    W = {}
    def walk(v, w):   # path weights from S
        W[v] = W.get(v, 0.0) + w
        for p, c, wt in g.edges:
            if p == v:
                walk(c, w * wt)
    walk(0, 1.0)
    assert all(abs(W[L] - 1.0) < 1e-12 for L in g.leaves())
    assert any(w == 0.5 for _, _, w in g.edges) or ni < 4   # shared children present


def test_oracle_on_wide_dag_keeps_simplex():
    base = P.config("C3")
    cfg = dataclasses.replace(base, name="W", kind="wide", wide_ni=8, classes=12, seed=108, nx=12, ny=10, nz=6,
                              n_shapes=36)
    inp = P.generate(cfg)
    u, q = O.run_inputs(inp, 20)
    assert np.max(np.abs(u.sum(axis=0) - 1.0)) < 1e-12 and np.min(u) >= 0.0
