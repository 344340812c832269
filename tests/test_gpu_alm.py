"""Explicit-flow ALM comparison arm (pf_config.method = PF_METHOD_EXPLICIT_ALM) against
the independent oracle oracle/alm.py potts_alm (fp64), same seeded inputs, same iteration count."""
import numpy as np
import pytest

import oracle as O
import paper_1501_07844_b200 as pf
import phantoms as P
from helpers import bf16_rounded, compare, solver_from_inputs
from oracle import alm as A

pytestmark = pytest.mark.gpu

CA, TA = 0.3, 0.11


def _oracle(inp, n, cap):
    K = inp.D.shape[0]
    if inp.s_kind == "shared_field":
        S = np.repeat(inp.s_field[None].astype(np.float64), K, axis=0)
    else:
        S = np.stack([np.full(inp.shape, float(inp.s_scalars[1 + l])) for l in range(K)])
    return A.potts_alm(inp.D, S, inp.cfg.ndim, n, ca=CA, ta=TA, cap=cap)


@pytest.mark.parametrize("name,dims,n,cap", [
    ("C1", (64, 64, 1), 150, "l2"),
    ("C2", (37, 29, 21), 100, "l2"),       # ragged tiles / z-chunks, edge-weighted shared S field
    ("C5", (24, 20, 40), 60, "l2"),        # K = 16, two z-chunks
    ("C1", (40, 33, 1), 120, "linf"),
    ("C2bf16", (30, 22, 17), 80, "l2"),    # D stored as bf16: the ALM solves the problem with bf16(D) too
])
def test_alm_matches_oracle(name, dims, n, cap):
    bf16 = name.endswith("bf16")
    inp = P.generate(P.config(name.replace("bf16", "")).resized(*dims))
    if bf16:
        inp = bf16_rounded(inp)
    s = solver_from_inputs(inp, method=pf.PF_METHOD_EXPLICIT_ALM, c=CA, tau=TA, cap=0 if cap == "l2" else 1,
                           d_bf16=bf16)
    s.iterate(n)
    u, am = s.labeling()
    q = s.flows()
    s.close()
    ur, qr, _ = _oracle(inp, n, cap)
    compare(u, q, ur, qr)
    assert np.array_equal(am, O.argmax(u))


def test_alm_and_pseudo_flow_reach_the_same_labeling():
    """Both methods solve the same convex relaxation (Eq. 1 / Eq. 3): at convergence the thresholded
    labelings agree and the energies match (the paper's claim that the pseudo-flow needs less memory
    is only meaningful because of this)."""
    inp = P.generate(P.config("C1").resized(48, 40, 1))
    a = solver_from_inputs(inp, method=pf.PF_METHOD_EXPLICIT_ALM, c=CA, tau=TA)
    b = solver_from_inputs(inp)
    a.iterate(6000)
    b.iterate(6000)
    ua, ama = a.labeling()
    ub, amb = b.labeling()
    ea, eb = a.energy(), b.energy()
    assert float(np.mean(ama == amb)) >= 0.999
    assert abs(ea[0] - eb[0]) <= 1e-3 * abs(eb[0])
    a.close()
    b.close()


@pytest.mark.parametrize("name,dims,n", [("C3", (33, 29, 17), 80), ("C4", (30, 26, 21), 80), ("C3", (40, 40, 12), 60)])
def test_dag_alm_matches_oracle(name, dims, n):
    """Explicit-flow ALM on HMF / DAGMF (Eq. 11): every node stores u_v, p_v and q_v."""
    inp = P.generate(P.config(name).resized(*dims))
    g = inp.graph
    s = solver_from_inputs(inp, method=pf.PF_METHOD_EXPLICIT_ALM, c=CA, tau=0.05)
    s.iterate(n)
    u, am = s.labeling()
    q = s.flows()
    s.close()
    S = np.stack([np.full(inp.shape, float(inp.s_scalars[v])) for v in range(g.num_nodes)])
    ur, qr, _ = A.dag_alm(inp.D, S, g.num_nodes, g.parent, g.child, g.weight, inp.cfg.ndim, n, ca=CA, ta=0.05)
    compare(u, q, ur, qr)


def test_alm_rejects_unsupported():
    inp = P.generate(P.config("I2").resized(20, 20, 8))   # Ishikawa chain (Alg. 3): not an Eq. 3 / Eq. 11 arm
    with pytest.raises(pf.PFError) as ei:
        solver_from_inputs(inp, method=pf.PF_METHOD_EXPLICIT_ALM)
    assert ei.value.status == pf.PF_ERR_UNSUPPORTED
    inp = P.generate(P.config("C2").resized(20, 20, 8))
    with pytest.raises(pf.PFError) as ei:
        solver_from_inputs(inp, method=pf.PF_METHOD_EXPLICIT_ALM, slab=(0, 4))
    assert ei.value.status == pf.PF_ERR_UNSUPPORTED
    s = solver_from_inputs(inp, method=pf.PF_METHOD_EXPLICIT_ALM)
    with pytest.raises(pf.PFError) as ei:
        s.iterate_phase(0)
    assert ei.value.status == pf.PF_ERR_UNSUPPORTED
    s.close()
