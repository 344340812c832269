"""z-slab decomposition on one GPU (row e): P consecutive slab solvers exchanging halo planes with
pf_exchange_local reproduce the single-domain solver BIT FOR BIT (every voxel's arithmetic is a
pure function of its neighbourhood)."""
import numpy as np
import pytest

import paper_1501_07844_b200 as pf
import phantoms as P
from helpers import solver_from_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["staged", "global"], autouse=True)
def kernel_variant(request, monkeypatch):
    """Run every test against both iteration kernels (TMA-staged default, global-load variant)."""
    monkeypatch.setenv("PF_ITER_KERNEL", request.param)
    return request.param


@pytest.mark.parametrize("phased", [False, True, "fused"])
@pytest.mark.parametrize("name,dims,parts", [("C2", (48, 40, 36), 2), ("C2", (48, 40, 37), 3), ("C4", (40, 33, 29), 4),
                                             ("C3", (33, 30, 24), 8), ("C5", (36, 33, 20), 5),
                                             ("C2", (40, 33, 9), 9)])   # one-plane slabs
def test_slabs_bitwise_equal_single_domain(name, dims, parts, phased):
    """phased: every iteration as pf_iterate_phase 0 (boundary planes) + 1 (interior), the multi-GPU
    overlap schedule."""
    cfg = P.config(name).resized(*dims)
    inp = P.generate(cfg)
    ref = solver_from_inputs(inp)
    ref.iterate(25)
    u_ref, a_ref = ref.labeling()
    q_ref = ref.flows()
    e_ref = ref.energy()
    solvers = [solver_from_inputs(inp, slab=b) for b in pf.solver.slab_bounds(cfg.nz, parts)]
    if phased == "fused":
        if not all(s.kernel_info()["staged"] for s in solvers):
            pytest.skip("fused halo stores need the TMA-staged kernels")
        slabs = pf.SlabSet(solvers, fused=True)
    else:
        slabs = pf.SlabSet(solvers, phased=phased)
    slabs.iterate(25)
    u, a = slabs.labeling()
    q = slabs.flows()
    assert np.array_equal(u, u_ref) and np.array_equal(a, a_ref) and np.array_equal(q, q_ref)
    e = slabs.energy()
    assert abs(e[0] - e_ref[0]) <= 1e-9 * abs(e_ref[0]) and abs(e[1] - e_ref[1]) <= 1e-9 * abs(e_ref[0])
    slabs.close()
    ref.close()


def test_phase_order_errors():
    cfg = P.config("C2").resized(40, 33, 12)
    inp = P.generate(cfg)
    s = solver_from_inputs(inp, slab=(4, 8))
    with pytest.raises(pf.PFError) as ei:
        s.iterate_phase(1)
    assert ei.value.status == pf.PF_ERR_STATE
    s.iterate_phase(0)
    with pytest.raises(pf.PFError) as ei:
        s.iterate(1)
    assert ei.value.status == pf.PF_ERR_STATE
    with pytest.raises(pf.PFError) as ei:
        s.iterate_phase(0)
    assert ei.value.status == pf.PF_ERR_STATE
    with pytest.raises(pf.PFError) as ei:
        s.iterate_phase(2)
    assert ei.value.status == pf.PF_ERR_INVALID
    s.iterate_phase(1)
    assert s.iterations() == 1
    s.close()


def test_linked_slab_rules(monkeypatch):
    """Linked slabs iterate only through pf_iterate_linked; kernel variants without whole-tile stores
    refuse to link (they keep pf_exchange_local)."""
    cfg = P.config("C2").resized(40, 33, 12)
    inp = P.generate(cfg)
    if solver_from_inputs(inp).kernel_info()["staged"]:
        ss = [solver_from_inputs(inp, slab=b) for b in pf.solver.slab_bounds(cfg.nz, 2)]
        pf.pf_link_slabs([s.h for s in ss])
        for s in ss:
            with pytest.raises(pf.PFError) as ei:
                s.iterate(1)
            assert ei.value.status == pf.PF_ERR_STATE
        pf.pf_iterate_linked([s.h for s in ss], 3)
        assert all(s.iterations() == 3 for s in ss)
        for s in ss:
            s.close()
    monkeypatch.setenv("PF_ITER_KERNEL", "global")
    ss = [solver_from_inputs(inp, slab=b) for b in pf.solver.slab_bounds(cfg.nz, 2)]
    with pytest.raises(pf.PFError) as ei:
        pf.pf_link_slabs([s.h for s in ss])
    assert ei.value.status == pf.PF_ERR_UNSUPPORTED
    for s in ss:
        s.close()


@pytest.mark.parametrize("fused", [False, True])
def test_slab_resume_from_single_domain_state(fused):
    """Checkpoint of a single-domain run restored into a slab set (pf_set_state per slab + one halo
    exchange): the continued slab run equals the uninterrupted single-domain run, bitwise."""
    cfg = P.config("C2").resized(40, 33, 23)
    inp = P.generate(cfg)
    ref = solver_from_inputs(inp)
    ref.iterate(17)
    u, q, it = ref.state()
    ref.iterate(14)
    solvers = [solver_from_inputs(inp, slab=b) for b in pf.solver.slab_bounds(cfg.nz, 3)]
    if fused and not all(s.kernel_info()["staged"] for s in solvers):
        pytest.skip("fused halo stores need the TMA-staged kernels")
    slabs = pf.SlabSet(solvers, fused=fused)
    slabs.iterate(3)                     # some other state first
    slabs.set_state(u, q, it)
    slabs.iterate(14)
    u2, q2, it2 = slabs.state()
    assert it2 == it + 14
    assert np.array_equal(u2, ref.state()[0]) and np.array_equal(q2, ref.flows())
    assert np.array_equal(slabs.labeling()[0], ref.labeling()[0])
    slabs.close()
    ref.close()


def test_phase1_grid_leaves_sms_free_for_the_exchange(kernel_variant):
    """pf_set_reserved_sms: the interior launch of a split iteration (pf_iterate_phase(1)) leaves SMs free for
    a concurrent exchange kernel (DistSolver reserves 8 for NCCL's P2P kernel); results stay bitwise equal."""
    import torch
    if kernel_variant != "staged":
        pytest.skip("the phase split and its persistent grid belong to the TMA-staged kernel")
    cfg = P.config("C2").resized(256, 256, 24)     # >= 148 work items per phase-1 launch
    inp = P.generate(cfg)
    bounds = pf.solver.slab_bounds(cfg.nz, 2)
    plain = pf.SlabSet([solver_from_inputs(inp, slab=b) for b in bounds], phased=True)
    resv = pf.SlabSet([solver_from_inputs(inp, slab=b) for b in bounds], phased=True)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for s in resv.solvers:
        s.set_reserved_sms(8)
        k = s.kernel_info()
        assert k["staged"] == 1
        assert 0 < k["phase1_ctas"] <= (sms - 8) * k["ctas_per_sm"] < k["ctas"]
    for s in plain.solvers:
        assert s.kernel_info()["phase1_ctas"] == s.kernel_info()["ctas"]
    plain.iterate(12)
    resv.iterate(12)
    assert np.array_equal(plain.labeling()[0], resv.labeling()[0]) and np.array_equal(plain.flows(), resv.flows())
    with pytest.raises(pf.PFError):
        resv.solvers[0].set_reserved_sms(sms)
    plain.close()
    resv.close()
