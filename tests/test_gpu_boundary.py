"""The C-ABI contract on the GPU (-m gpu): plans independent of each other,
argument validation of the binding's output buffers, the geometry-keyed filter
bank (lt_bank_key / lt_set_bank / lt_save_bank / lt_load_bank), and the
library-owned combine (lt_combine_rois with an NCCL communicator)."""
import math
import os

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def relerr(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def lt():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1604_02292_b200 as m
    assert torch.cuda.is_available()
    return m


def test_two_plans_one_device_different_nfgp(lt, orc):
    """Two plans on one device, interleaved, with different n_FGP (and ROI
    sizes): each matches the oracle (<= 1e-3) and its own isolated solve
    bitwise (no state shared through per-process tables)."""
    inp = synth.make_inputs("C1")
    p = inp.sino.astype(np.float64)
    n_iter = 6
    a = lt.Plan(64, inp.angles, 91, [[32, 32]], 12, 8, n_iter)
    b = lt.Plan(64, inp.angles, 91, [[20, 40], [40, 24]], 8, 6, n_iter)
    sino = torch.from_numpy(inp.sino).cuda()
    a.filter_bank(); b.filter_bank()
    ra1 = a.tv_solve(sino, 0.05, 7).cpu().numpy()
    rb1 = b.tv_solve(sino, 0.02, 31).cpu().numpy()
    ra2 = a.tv_solve(sino, 0.05, 7).cpu().numpy()
    rb2 = b.tv_solve(sino, 0.02, 31).cpu().numpy()
    assert np.array_equal(ra1, ra2) and np.array_equal(rb1, rb2)
    oa = orc.pipeline(p, inp.angles, 64, [[32, 32]], 12, 8, n_iter, mode="tv", lam=0.05, n_fgp=7)
    ob = orc.pipeline(p, inp.angles, 64, [[20, 40], [40, 24]], 8, 6, n_iter, mode="tv", lam=0.02, n_fgp=31)
    assert relerr(ra1[0], oa[0]) <= 1e-3
    for q, g in enumerate(b.local_rois):
        assert relerr(rb1[q], ob[g]) <= 1e-3


def test_output_buffer_validation(lt):
    inp = synth.make_inputs("C1")
    plan = lt.Plan(64, inp.angles, 91, inp.centres, 12, 8, 3)
    plan.filter_bank()
    sino = torch.from_numpy(inp.sino).cuda()
    good = torch.empty(1, 24, 24, device="cuda")
    plan.sirt_solve(sino, out=good)
    with pytest.raises(ValueError):
        plan.sirt_solve(sino, out=torch.empty(1, 24, 23, device="cuda"))          # wrong shape
    with pytest.raises(TypeError):
        plan.sirt_solve(sino, out=torch.empty(1, 24, 24, device="cuda", dtype=torch.float64))
    with pytest.raises(ValueError):
        plan.sirt_solve(sino, out=torch.empty(1, 24, 48, device="cuda")[:, :, ::2])   # strided view
    with pytest.raises(TypeError):
        plan.sirt_solve(sino, out=torch.empty(1, 24, 24))                           # host tensor
    with pytest.raises(ValueError):
        plan.sirt_solve(sino[:, :90].contiguous())                                  # wrong sinogram size
    with pytest.raises(ValueError):
        plan.combine(torch.empty(1, 24, 24, device="cuda"), [0], out=torch.empty(64, 63, device="cuda"))
    with pytest.raises(ValueError):
        plan.solve_host("sirt", torch.from_numpy(inp.sino), 0.0, math.inf, image_host=torch.empty(63, 64))


def test_bank_key_set_save_load(lt, tmp_path):
    inp = synth.make_inputs("C1")
    n_iter = 12
    a = lt.Plan(64, inp.angles, 91, inp.centres, 12, 8, n_iter)
    a.filter_bank()
    sino = torch.from_numpy(inp.sino).cuda()
    ref = a.sirt_solve(sino).cpu().numpy()
    path = str(tmp_path / "c1.bank")
    a.save_bank(path)
    # same geometry, fewer iterations and other ROIs: the first n filters are reused
    b = lt.Plan(64, inp.angles, 91, inp.centres, 12, 8, n_iter)
    b.load_bank(path)
    assert np.array_equal(b.sirt_solve(sino).cpu().numpy(), ref)
    c = lt.Plan(64, inp.angles, 91, [[20, 20]], 6, 4, 5)
    c.load_bank(path)
    assert torch.equal(c.get_bank(), a.get_bank()[:5])
    assert c.bank_key == a.bank_key
    # another geometry: rejected by key
    other = lt.Plan(64, inp.angles[:-1], 91, inp.centres, 12, 8, n_iter)
    assert other.bank_key != a.bank_key
    with pytest.raises(ValueError):
        other.load_bank(path)
    with pytest.raises(ValueError):
        lt.Plan(64, inp.angles, 91, inp.centres, 12, 8, n_iter + 1).load_bank(path)   # too few filters
    with pytest.raises(ValueError):
        other.set_bank(a.get_bank()[:, :-1].contiguous(), key=a.bank_key)
    other.set_bank(torch.zeros(n_iter, len(inp.angles) - 1, 91, device="cuda"), key=other.bank_key)
    not_a_bank = tmp_path / "x.bank"
    not_a_bank.write_bytes(b"hello world" * 10)
    with pytest.raises(ValueError):
        b.load_bank(str(not_a_bank))


def test_combine_rois_library_owned_world1(lt):
    """lt_combine_rois on one rank: without a communicator and with a 1-rank
    NCCL communicator (lt_nccl_comm_init) it equals the stitch of the cores."""
    cfg = synth.config("C2")
    inp = synth.make_inputs("C2")
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, 4)
    plan.filter_bank()
    cores = plan.sirt_solve(torch.from_numpy(inp.sino).cuda())
    ref = plan.combine(cores, plan.local_rois)
    got0 = plan.combine_rois(cores)
    comm = lt.NcclComm(1, 0, lt.NcclComm.unique_id())
    try:
        got1 = plan.combine_rois(cores, comm)
    finally:
        comm.close()
    assert torch.equal(got0, ref) and torch.equal(got1, ref)
    spr, table = plan.slot_table()
    assert spr == plan.R and np.array_equal(table, plan.local_rois)
