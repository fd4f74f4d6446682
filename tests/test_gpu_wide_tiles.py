"""Extended ROIs wider than 256 px (up to 320: the paper's 256^2 local parts
padded by 1/8 of their size per side) on the fast
kernels (-m gpu): the 10-columns-per-lane FGP clusters (k_fgp2 CP = 5), the
wide forward projector (336-entry staged lines, 15 rays per lane) and the
backprojector, against the fp64 oracle."""
import math

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


@pytest.mark.parametrize("h,w", [(320, 320), (257, 319), (300, 262), (64, 320)])
def test_fgp_wide_tiles(lt, orc, h, w):
    """FGP prox (Beck & Teboulle; A13) on tiles wider / taller than 256."""
    rng = np.random.default_rng(h * 1000 + w)
    x = rng.random((2, h, w)).astype(np.float32)
    got = lt.fgp_batch(torch.from_numpy(x).cuda(), 0.05, 30).cpu().numpy()
    for i in range(2):
        assert relerr(got[i], orc.fgp(x[i].astype(np.float64), 0.05, 30)) <= 1e-5, (h, w, i)


def _wide_geometry():
    n, na = 512, 96
    nd = int(math.ceil(math.sqrt(2) * n)) | 1
    ang = synth.angles_for(na)
    cen = np.array([[256, 256], [128, 384], [384, 130]], dtype=np.int32)   # central, clipped top-right / bottom-left
    return n, na, nd, ang, cen, 128, 32


def test_wide_roi_project_backproject_all_bins(lt, orc):
    """W_{L'} x on ALL bins and M_{L'} W^T s for 320-wide extended ROIs."""
    n, na, nd, ang, cen, r, m = _wide_geometry()
    plan = lt.Plan(n, ang, nd, cen, r, m, 1)
    assert plan.h == 160
    rects = orc.roi_rects(n, cen, r, m)
    rng = np.random.default_rng(7)
    x = rng.random((n, n)); s = rng.standard_normal((na, nd))
    xg = torch.from_numpy(x.astype(np.float32)).cuda(); sg = torch.from_numpy(s.astype(np.float32)).cuda()
    for q in range(plan.R):
        g = int(plan.local_rois[q])
        rect = tuple(int(v) for v in rects[g][4:8])
        ref = orc.forward(x, ang, nd, rect)
        got = plan.project(xg, roi=q).cpu().double().numpy()
        assert relerr(got, ref) <= 1e-5, q
        assert np.all(got[ref == 0] == 0)
        refb = orc.back(s, ang, n, rect)
        assert relerr(plan.backproject(sg, roi=q).cpu().double().numpy(), refb) <= 1e-5, q


def test_wide_tv_solve_matches_oracle(lt, orc):
    """Local FISTA-TV (Alg. 3) on 320-wide extended ROIs, central and
    clipped, disc on: every core <= 1e-3 against the oracle's pipeline."""
    n, na, nd, ang, cen, r, m = _wide_geometry()
    shapes = synth.random_shapes(n, 12, 6, np.random.default_rng(3))
    p = synth.analytic_sinogram(shapes, ang, nd)
    p = (p + np.random.default_rng(4).normal(0, 0.01 * p.max(), p.shape)).astype(np.float32)
    n_iter, lam, nf = 8, 0.05, 30
    plan = lt.Plan(n, ang, nd, cen, r, m, n_iter)
    plan.filter_bank()
    cores = plan.tv_solve(torch.from_numpy(p).cuda(), lam, nf).cpu().numpy()
    ref = orc.pipeline(p.astype(np.float64), ang, n, cen, r, m, n_iter, mode="tv", lam=lam, n_fgp=nf)
    for q, g in enumerate(plan.local_rois):
        assert relerr(cores[q], ref[g]) <= 1e-3, g
    # box mode on the same wide tiles
    sb = plan.sirt_solve(torch.from_numpy(p).cuda(), 0.0, math.inf).cpu().numpy()
    refb = orc.pipeline(p.astype(np.float64), ang, n, cen, r, m, n_iter, mode="box")
    for q, g in enumerate(plan.local_rois):
        assert relerr(sb[q], refb[g]) <= 1e-3, g


def test_p1_config_plan(lt):
    """The paper's experiment geometry (config P1) plans onto the fast kernels:
    one 320 x 320 extended ROI, TV accepted (before: error 2 above 256)."""
    cfg = synth.config("P1")
    inp = synth.make_inputs("P1")
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, 3)
    plan.filter_bank()
    cores = plan.tv_solve(torch.from_numpy(inp.sino).cuda(), cfg.lam, 10)
    assert cores.shape == (1, 256, 256) and torch.isfinite(cores).all()
