"""Temporal blocking (pf_config.tblock = 2): two iterations of the pseudo-flow while-loop per HBM
pass.  Every per-point step is the one-iteration kernels' arithmetic in the same order, so a tblock solver is
BITWISE a tblock = 0 solver (fields, labeling, residuals), and through it the oracle parity carries over; one
oracle case is checked directly."""
import numpy as np
import pytest

import oracle as O
import phantoms as P
from helpers import compare, solver_from_inputs

pf = pytest.importorskip("paper_1501_07844_b200")

pytestmark = pytest.mark.gpu


def _cfg(K, dims, sfield=True, seed=2020):
    nx, ny, nz = dims
    ndim = 2 if nz == 1 else 3
    return P.Config(f"T{K}", ndim, nx, ny, nz, "potts", K, 4 * K, 0.15, "sq", "edge" if sfield else "scalar",
                    0.05 if sfield else 0.1, 300, seed=seed)


def _pair(inp, n, **kw):
    a = solver_from_inputs(inp, **kw)
    b = solver_from_inputs(inp, tblock=2, **kw)
    assert b.kernel_info()["tblock"] == 2 and a.kernel_info()["tblock"] == 1
    ra = a.iterate(n, residual=True)
    rb = b.iterate(n, residual=True)
    out = (a.labeling(), a.flows(), ra, b.labeling(), b.flows(), rb)
    a.close()
    b.close()
    return out


@pytest.mark.parametrize("K,dims,n,shift,cap,sfield", [
    (4, (64, 48, 40), 30, 0, 0, True),      # several z-chunks, shared S field
    (4, (67, 45, 37), 31, 1, 0, True),      # ragged x (28-wide tiles), y, z; odd n: one plain iteration at the end
    (3, (57, 33, 29), 20, 0, 1, False),     # l-inf boxes, scalar capacities
    (2, (30, 20, 10), 25, 0, 0, True),
    (4, (97, 41, 1), 40, 0, 0, True),       # 2-D
    (3, (29, 9, 2), 12, 0, 0, True),        # two planes
    (2, (5, 3, 70), 16, 1, 0, False),       # a deep, thin column
])
def test_tblock_bitwise_equals_one_iteration_per_pass(K, dims, n, shift, cap, sfield):
    inp = P.generate(_cfg(K, dims, sfield))
    (ua, la), qa, ra, (ub, lb), qb, rb = _pair(inp, n, shift=shift, cap=cap)
    assert np.array_equal(ua, ub) and np.array_equal(la, lb) and np.array_equal(qa, qb)
    assert ra == rb


@pytest.mark.parametrize("check_every", [1, 3, 10])
def test_tblock_residual_positions(check_every):
    """The residual of the pair's last check iteration (first or second iteration of a pair), any cadence."""
    inp = P.generate(_cfg(3, (40, 30, 20)))
    for n in (2, 3, 7, 10):
        a = solver_from_inputs(inp, check_every=check_every)
        b = solver_from_inputs(inp, check_every=check_every, tblock=2)
        assert a.iterate(n, residual=True) == b.iterate(n, residual=True)
        a.close()
        b.close()


def test_tblock_oracle_parity(  ):
    """300 iterations of a 4-label C2-recipe volume against the paper-exact oracle."""
    inp = P.generate(_cfg(4, (64, 64, 48)))
    s = solver_from_inputs(inp, tblock=2)
    s.iterate(300)
    u, am = s.labeling()
    q = s.flows()
    s.close()
    ur, qr = O.run_inputs(inp, 300)
    compare(u, q, ur, qr)
    assert np.array_equal(am, np.argmax(u, 0).astype(np.uint8))


def test_tblock_unsupported():
    with pytest.raises(pf.PFError):   # 8 labels: the on-chip state of K > 4 does not fit
        solver_from_inputs(P.generate(P.config("C2").resized(40, 30, 20)), tblock=2)
    with pytest.raises(pf.PFError):   # DAG
        solver_from_inputs(P.generate(P.config("C4").resized(40, 30, 20)), tblock=2)
    with pytest.raises(pf.PFError):   # slabs
        solver_from_inputs(P.generate(_cfg(3, (40, 30, 20))), tblock=2, slab=(0, 10))
    with pytest.raises(pf.PFError):
        solver_from_inputs(P.generate(_cfg(3, (40, 30, 20))), tblock=3)
