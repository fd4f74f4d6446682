"""Out-of-bounds and race checks of our own (-m gpu).  compute-sanitizer is not
available on the GPU pool, so every workspace region of a
LT_GUARD_BANDS plan is followed by a canary band that lt_guard_check compares
after the solves: a kernel writing past its region (any launch shape: band-split
projector, angle-split backprojector partials, persistent FGP clusters, the
stitch, the global solvers) damages a band.  Races (mbarrier phases, DSMEM
hand-over, cp.async double buffering) would make repeated solves differ, so the
split and persistent launch shapes are also repeated and compared bitwise."""
import math

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lt():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1604_02292_b200 as m
    assert torch.cuda.is_available()
    return m


def _assert_intact(plan):
    bad, off = plan.guard_check()
    assert bad == 0, f"{bad} canary bands damaged, first at workspace byte {off}"


def test_guard_bands_detect_a_stray_write(lt):
    """Negative control: a byte written into the last canary band is reported."""
    inp = synth.make_inputs("C1")
    plan = lt.Plan(64, inp.angles, 91, inp.centres, 12, 8, 2, guard_bands=True)
    _assert_intact(plan)
    plan.ws[plan.workspace_bytes - 7] = 0
    bad, off = plan.guard_check()
    assert bad == 1 and off == plan.workspace_bytes - 7


@pytest.mark.parametrize("case", ["C1", "C2"])
def test_guard_bands_small_configs_every_entry(lt, case):
    cfg = synth.config(case)
    inp = synth.make_inputs(case)
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, 3, guard_bands=True)
    plan.filter_bank()
    sino = torch.from_numpy(inp.sino).cuda()
    c1 = plan.sirt_solve(sino, 0.0, math.inf)
    c2 = plan.tv_solve(sino, 0.05, 5)
    plan.tv_solve(sino, np.linspace(0.0, 0.1, plan.R), 4)
    plan.haar_solve(sino, 0.02, 3 if case == "C1" else 0)     # (C2 has clipped ROIs: 0 levels)
    plan.exterior_solve(sino)
    plan.combine(c2, plan.local_rois)
    plan.combine_rois(c2)
    plan.get_ext()
    x = torch.rand(cfg.n, cfg.n, device="cuda")
    plan.project(x); plan.backproject(sino); plan.project(x, roi=0); plan.backproject(sino, roi=0)
    plan.disc_correct(sino)
    plan.global_sirt(sino, 2); plan.global_tv(sino, 2, 0.05, 3); plan.global_cp(sino, 2, 10.0)
    plan.solve_host("tv", torch.from_numpy(inp.sino), 0.05, 0.0, 4)
    torch.cuda.synchronize()
    _assert_intact(plan)
    assert torch.isfinite(c1).all() and torch.isfinite(c2).all()


def test_guard_bands_and_repeatability_split_launches(lt):
    """T1: one 256^2 ROI of a 1024^2 / 512-angle geometry -> band-split forward
    projector + join, angle-split backprojector (stage 1/2), 16-CTA FGP."""
    cfg = synth.config("T1")
    inp = synth.make_inputs("T1")
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, 4, guard_bands=True)
    plan.filter_bank()
    sino = lt.pad_truncated(torch.from_numpy(inp.sino_trunc).cuda(), cfg.n_det)
    ref = plan.tv_solve(sino, 0.05, 10).clone()
    for _ in range(4):
        assert torch.equal(plan.tv_solve(sino, 0.05, 10), ref)
    s_ref = plan.sirt_solve(sino, 0.0, math.inf).clone()
    assert torch.equal(plan.sirt_solve(sino, 0.0, math.inf), s_ref)
    _assert_intact(plan)


def test_guard_bands_and_repeatability_persistent_fgp(lt):
    """64 ROIs of the C4 geometry (256^2 tiles, > 3 waves of 8-CTA clusters):
    the persistent FGP (cp.async prefetch of the next tile, mbarrier
    invalidation / re-initialisation per tile) -- canaries intact and five
    repeated solves bitwise identical."""
    cfg = synth.config("C4")
    inp = synth.make_inputs("C4")
    cen = inp.centres[np.arange(0, 256, 4)]
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, cen, cfg.radius, cfg.margin, 3, guard_bands=True)
    plan.filter_bank()
    sino = torch.from_numpy(inp.sino).cuda()
    ref = plan.tv_solve(sino, 0.05, 20).clone()
    for _ in range(4):
        assert torch.equal(plan.tv_solve(sino, 0.05, 20), ref)
    _assert_intact(plan)
