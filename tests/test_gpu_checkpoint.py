"""Checkpoint / resume (SURVEY P11 "save/resume bitwise"; pf_set_state): a run of a + b iterations equals
a iterations, save, a NEW solver loaded from the checkpoint, b iterations -- bitwise, residual included."""
import numpy as np
import pytest

import phantoms as P
from helpers import solver_from_inputs

pf = pytest.importorskip("paper_1501_07844_b200")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,dims,a,b", [
    ("C2", (37, 29, 23), 150, 150),      # Potts, staged kernel, CUDA graphs on the long calls
    ("C4", (30, 26, 19), 60, 47),        # DAG with shared leaves
    ("I2", (33, 21, 17), 40, 33),        # Ishikawa (zero flows of the end labels are not stored)
    ("C5", (45, 37, 21), 30, 23),        # K = 16: the 2-CTA cluster kernel
])
def test_resume_equals_uninterrupted_run(name, dims, a, b, tmp_path):
    inp = P.generate(P.config(name).resized(*dims))
    ref = solver_from_inputs(inp)
    ref.iterate(a)
    path = str(tmp_path / "ck.npz")
    ref.save(path, c=inp.cfg.c, tau=inp.cfg.tau)
    r_ref = ref.iterate(b, residual=True)
    u_ref, lab_ref = ref.labeling()
    q_ref = ref.flows()

    res = solver_from_inputs(inp)
    res.iterate(7)                       # some other state first: load must replace all of it
    c, tau = res.load(path)
    assert (c, tau) == (inp.cfg.c, inp.cfg.tau)
    assert res.iterations() == a
    r_res = res.iterate(b, residual=True)
    u_res, lab_res = res.labeling()
    assert res.iterations() == a + b
    assert np.array_equal(u_ref, u_res) and np.array_equal(lab_ref, lab_res)
    assert np.array_equal(q_ref, res.flows())
    assert r_ref == r_res
    ref.close()
    res.close()


def test_set_state_from_device_buffers():
    import torch
    inp = P.generate(P.config("C2").resized(40, 24, 18))
    s1, s2 = solver_from_inputs(inp), solver_from_inputs(inp)
    s1.iterate(25)
    u, q, it = s1.state()
    s2.set_state(torch.from_numpy(u).cuda(), torch.from_numpy(q).cuda(), it)
    s1.iterate(12)
    s2.iterate(12)
    torch.cuda.synchronize()
    assert np.array_equal(s1.labeling()[0], s2.labeling()[0]) and np.array_equal(s1.flows(), s2.flows())


def test_set_state_linear_labeling_matches_oracle():
    """pf_set_state with the labeling u itself (u_is_log2 = 0): start from the oracle's state after 40
    iterations, run 60 more, compare with the oracle's 100 (the log2 conversion is the only extra rounding)."""
    import oracle as O
    from helpers import compare
    inp = P.generate(P.config("C4").resized(33, 27, 19))
    u40, q40 = O.run_inputs(inp, 40)
    s = solver_from_inputs(inp)
    s.set_state(u40.astype(np.float32), q40.astype(np.float32), 40, u_is_log2=False)
    s.iterate(60)
    u, _ = s.labeling()
    q = s.flows()
    O.run_inputs(inp, 60, state=(u40, q40))
    compare(u, q, u40, q40)
    s.close()


def test_dead_label_stays_dead():
    """A label set exactly to 0 (lambda = -inf) stays 0 -- the multiplicative update of Eq. 7 keeps
    u_L = 0 -- in the GPU state as in the oracle, and the other labels follow the oracle."""
    import oracle as O
    from helpers import compare
    inp = P.generate(P.config("C2").resized(29, 23, 17))
    ur, qr = O.init_state(8, 8, inp.shape, 3)
    ur[3] = 0.0
    ur /= ur.sum(0)
    s = solver_from_inputs(inp)
    s.set_state(ur.astype(np.float32), qr.astype(np.float32), 0, u_is_log2=False)
    s.iterate(50)
    u, am = s.labeling()
    O.run_inputs(inp, 50, state=(ur, qr))
    assert np.all(u[3] == 0) and np.all(ur[3] == 0) and not np.any(am == 3)
    compare(u, s.flows(), ur, qr)
    s.close()


def test_set_state_errors(tmp_path):
    inp = P.generate(P.config("C2").resized(20, 16, 8))
    s = solver_from_inputs(inp)
    u, q, _ = s.state()
    with pytest.raises(pf.PFError):
        pf.pf_set_state(s.h, None, q, 0)
    with pytest.raises(pf.PFError):
        s.set_state(u, q, -1)
    with pytest.raises(ValueError):               # validated sizes / dtypes in the binding (no silent misuse)
        s.set_state(u[:, :-1], q, 0)
    with pytest.raises(ValueError):
        s.set_state(u.astype(np.float64), q, 0)
    with pytest.raises(ValueError):
        s.labeling(u_out=np.empty((u.shape[0] - 1,) + u.shape[1:], np.float32))
    path = str(tmp_path / "ck.npz")
    s.save(path)
    other = solver_from_inputs(P.generate(P.config("C2").resized(20, 16, 9)))
    with pytest.raises(ValueError):
        other.load(path)
    alm = solver_from_inputs(inp, method=pf.PF_METHOD_EXPLICIT_ALM, c=0.3, tau=0.11)
    with pytest.raises(pf.PFError):
        alm.set_state(u, q, 0)
    for x in (s, other, alm):
        x.close()
