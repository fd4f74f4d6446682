"""GPU parity: the CUDA path (through the C-ABI binding) against the fp64
oracle on the same seeded inputs (-m gpu).

Tolerances (north star / DESIGN.md §Parity): one A or A^T application and the
convolution cache <= 1e-5 relative L2 (fp32); filter bank <= 1e-4; full solves
<= 1e-3 per ROI core and on the stitched image; ROI indexing exact.
"""
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


def nd_for(n):
    return int(math.ceil(math.sqrt(2) * n)) | 1


def gpu(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def cpu(t):
    torch.cuda.synchronize()
    return t.detach().cpu().double().numpy()


# ------------------------------------------------------------------ operators

@pytest.mark.parametrize("n,na,span", [(64, 32, math.pi), (300, 45, math.pi), (200, 32, 2 * math.pi / 3), (37, 17, math.pi)])
def test_global_project_backproject(lt, orc, n, na, span):
    nd = nd_for(n)
    ang = synth.angles_for(na, span)
    plan = lt.Plan(n, ang, nd, [[n // 2, n // 2]], 4, 2, 1)
    rng = np.random.default_rng(n)
    x = rng.random((n, n)); s = rng.standard_normal((na, nd))
    assert relerr(cpu(plan.project(gpu(x))), orc.forward(x, ang, nd)) <= 1e-5
    assert relerr(cpu(plan.backproject(gpu(s))), orc.back(s, ang, n)) <= 1e-5
    # fp32 adjoint identity on the GPU pair
    wx = cpu(plan.project(gpu(x))); wts = cpu(plan.backproject(gpu(s)))
    assert abs(np.vdot(wx, s) - np.vdot(x, wts)) <= 1e-5 * np.linalg.norm(wx) * np.linalg.norm(s)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_roi_project_backproject_all_bins(lt, orc, cfg):
    """W_{L'} x = W(M_{L'} x) on ALL bins (window correctness) and M_{L'} W^T s,
    for every ROI including clipped ones."""
    c = synth.config(cfg)
    ang = synth.angles_for(c.n_angles, c.span)
    cen = synth.roi_centres(c)[:6]
    cen = np.concatenate([cen, [[c.radius, c.radius], [c.n - c.radius, c.radius]]]).astype(np.int32)
    plan = lt.Plan(c.n, ang, c.n_det, cen, c.radius, c.margin, 1)
    rects = orc.roi_rects(c.n, cen, c.radius, c.margin)
    rng = np.random.default_rng(3)
    x = rng.random((c.n, c.n)); s = rng.standard_normal((c.n_angles, c.n_det))
    xg, sg = gpu(x), gpu(s)
    for q in range(plan.R):
        g = plan.local_rois[q]
        rect = tuple(int(v) for v in rects[g][4:8])
        ref = orc.forward(x, ang, c.n_det, rect)
        got = cpu(plan.project(xg, roi=q))
        assert relerr(got, ref) <= 1e-5, (cfg, q)
        assert np.all(got[ref == 0] == 0)
        refb = orc.back(s, ang, c.n, rect)
        gotb = cpu(plan.backproject(sg, roi=q))
        assert relerr(gotb, refb) <= 1e-5, (cfg, q)
        assert np.all(gotb[refb == 0] == 0)


def test_filter_bank(lt, orc):
    n, na, nd, nk = 64, 32, 91, 100
    ang = synth.angles_for(na)
    plan = lt.Plan(n, ang, nd, [[32, 32]], 12, 8, nk)
    plan.filter_bank()
    got = cpu(plan.get_bank())
    ref = orc.filter_bank(n, ang, nd, nk)
    for k in (0, 9, 49, 99):
        assert relerr(got[k], ref[k]) <= 1e-4, k


def test_filter_bank_odd_limited(lt, orc):
    n, na, nk = 45, 20, 12
    nd = nd_for(n)
    ang = synth.angles_for(na, 2 * math.pi / 3)
    plan = lt.Plan(n, ang, nd, [[22, 22]], 5, 3, nk)
    plan.filter_bank()
    got = cpu(plan.get_bank())
    ref = orc.filter_bank(n, ang, nd, nk)
    assert relerr(got, ref) <= 1e-4


def test_disc_and_conv_cache(lt, orc):
    inp = synth.make_inputs("C1")
    n, nd, nk = 64, 91, 30
    plan = lt.Plan(n, inp.angles, nd, inp.centres, 12, 8, nk)
    plan.filter_bank()
    pc_g, c_g = plan.disc_correct(gpu(inp.sino))
    pc_o, c_o, _, _ = orc.disc(inp.sino.astype(np.float64), inp.angles, n)
    assert abs(cpu(c_g)[0] - c_o) <= 1e-5 * abs(c_o)
    assert relerr(cpu(pc_g), pc_o) <= 1e-5
    # stage-wise: oracle bank + oracle p_c in, b_k out
    bank_o = orc.filter_bank(n, inp.angles, nd, nk)
    plan.set_bank(gpu(bank_o))
    b_g = cpu(plan.conv_cache(gpu(pc_o)))
    b_o = orc.conv_cache(bank_o, pc_o)
    for k in (0, 5, 29):
        assert relerr(b_g[k], b_o[k]) <= 1e-5, k


def test_conv_cache_wide_detector(lt, orc):
    """Several 512-tap chunks and a ragged tail (N_d = 1449)."""
    rng = np.random.default_rng(4)
    n, na, nd, nk = 1024, 3, 1449, 9
    ang = synth.angles_for(na)
    plan = lt.Plan(n, ang, nd, [[512, 512]], 8, 0, nk, disc=False)
    bank = rng.standard_normal((nk, na, nd)) * np.exp(-np.abs(np.arange(nd) - 724) / 50.0)
    p = rng.random((na, nd))
    plan.set_bank(gpu(bank))
    got = cpu(plan.conv_cache(gpu(p)))
    ref = orc.conv_cache(bank.astype(np.float32).astype(np.float64), p.astype(np.float32).astype(np.float64))
    assert relerr(got, ref) <= 1e-5


# ------------------------------------------------------------------ FGP

@pytest.mark.parametrize("h,w", [(6, 6), (40, 40), (100, 77), (128, 128), (192, 192), (256, 256), (1, 9)])
def test_fgp_batch(lt, orc, h, w):
    rng = np.random.default_rng(h * 1000 + w)
    cnt = 3
    b = rng.random((cnt, h, w))
    lam, nf = 0.05, 100
    got = cpu(lt.fgp_batch(gpu(b), lam, nf))
    for q in range(cnt):
        ref = orc.fgp(b[q].astype(np.float32).astype(np.float64), lam, nf)
        assert relerr(got[q], ref) <= 1e-5, (h, w, q)


@pytest.mark.parametrize("cnt", [17, 32])
def test_fgp_batch_split_tail(lt, orc, cnt):
    """256-row tiles in batches with a ragged last wave of 8-CTA clusters
    (17 = 15 + 2, 32 = 2 x 15 + 2 co-resident clusters on B200): the first and
    last tiles against the oracle."""
    rng = np.random.default_rng(4000 + cnt)
    b = rng.random((cnt, 256, 240))
    lam, nf = 0.05, 30
    got = cpu(lt.fgp_batch(gpu(b), lam, nf))
    for q in list(range(3)) + list(range(cnt - 3, cnt)):
        ref = orc.fgp(b[q].astype(np.float32).astype(np.float64), lam, nf)
        assert relerr(got[q], ref) <= 1e-5, q


def test_fgp_lambda_zero_identity(lt):
    x = torch.rand(2, 30, 30, device="cuda")
    assert torch.equal(lt.fgp_batch(x, 0.0, 10), x)


# ------------------------------------------------------------------ full solves

def _oracle_solve(orc, inp, cfg, n_iter, mode, lam=0.0, nfgp=100, roi_idx=None, bank=None):
    cen = inp.centres if roi_idx is None else inp.centres[roi_idx]
    return orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, cen, cfg.radius, cfg.margin, n_iter,
                        mode=mode, lam=lam, n_fgp=nfgp, bank=bank, want_ext=True)


def test_sirt_solve_C1(lt, orc):
    cfg = synth.config("C1")
    inp = synth.make_inputs("C1")
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, cfg.n_iter)
    plan.filter_bank()
    cores = cpu(plan.sirt_solve(gpu(inp.sino), 0.0, math.inf))
    ext = cpu(plan.get_ext())
    ref, ref_ext = _oracle_solve(orc, inp, cfg, cfg.n_iter, "box")
    assert relerr(cores, ref) <= 1e-3
    assert relerr(ext, ref_ext) <= 1e-3
    assert cores.min() >= 0.0


def test_single_roi_split_launches(lt, orc):
    """One 256x256 extended ROI with 192 angles (the T1 shape at fewer angles and
    iterations): fewer CTAs than SMs, so the ROI forward projector splits its
    bands and the backprojections their angles (two-pass, ordered sums)."""
    cfg = synth.Config(22, "single-split", 384, 192, math.pi, 545, "poisson", 1e4, 1, 96, 32, "centre", 6,
                       "tv", 0.05, 20, 5, 0)
    inp = synth.make_inputs(cfg)
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, cfg.n_iter)
    plan.filter_bank()
    cores = cpu(plan.sirt_solve(gpu(inp.sino), 0.0, math.inf))
    ref, _ = _oracle_solve(orc, inp, cfg, cfg.n_iter, "box")
    assert relerr(cores, ref) <= 1e-3
    cores = cpu(plan.tv_solve(gpu(inp.sino), cfg.lam, cfg.n_fgp))
    ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, inp.centres, cfg.radius, cfg.margin,
                       cfg.n_iter, mode="tv", lam=cfg.lam, n_fgp=cfg.n_fgp)
    assert relerr(cores[0], ref[0]) <= 1e-3


def test_tv_solve_small(lt, orc):
    cfg = synth.Config(20, "tvsmall", 128, 24, math.pi, 181, "poisson", 1e4, 5, 16, 16, "seeded", 12, "tv",
                       0.05, 50, 6, 0)
    inp = synth.make_inputs(cfg)
    # the last two are clipped with valid rectangles at odd offsets (vr0 = 13, vc0 = 9;
    # vc0 = 15 with 51 valid rows): the FGP epilogue's scalar (unaligned) load / store paths
    cen = np.array([[64, 64], [16, 16], [112, 40], [40, 112], [20, 100], [19, 23], [109, 17]], dtype=np.int32)
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, cen, cfg.radius, cfg.margin, cfg.n_iter)
    plan.filter_bank()
    cores = cpu(plan.tv_solve(gpu(inp.sino), cfg.lam, cfg.n_fgp))
    ext = cpu(plan.get_ext())
    ref, ref_ext = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, cen, cfg.radius, cfg.margin,
                                cfg.n_iter, mode="tv", lam=cfg.lam, n_fgp=cfg.n_fgp, want_ext=True)
    for q in range(len(cen)):
        assert relerr(cores[q], ref[q]) <= 1e-3, q
    assert relerr(ext, ref_ext) <= 1e-3


def test_sirt_solve_C3_subset(lt, orc):
    """C3 geometry (limited angle [0, 2pi/3)), seeded ROIs, 30 iterations."""
    cfg = synth.config("C3")
    inp = synth.make_inputs("C3")
    n_iter = 30
    cen = inp.centres[:6]
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, cen, cfg.radius, cfg.margin, n_iter)
    plan.filter_bank()
    cores = cpu(plan.sirt_solve(gpu(inp.sino), 0.0, math.inf))
    ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, cen, cfg.radius, cfg.margin, n_iter,
                       mode="box")
    for q in range(len(cen)):
        assert relerr(cores[q], ref[q]) <= 1e-3, q


def test_combine_matches_oracle_stitch(lt, orc):
    n, r = 96, 8
    cen = np.array([[8, 8], [8, 24], [20, 30], [88, 88], [50, 50], [52, 54]], dtype=np.int32)
    plan = lt.Plan(n, synth.angles_for(4), nd_for(n), cen, r, 2, 1)
    cores = np.random.default_rng(5).random((6, 16, 16))
    got = cpu(plan.combine(gpu(cores), list(range(6))))
    ref = orc.stitch(n, cen, r, cores.astype(np.float32).astype(np.float64))
    assert relerr(got, ref) <= 1e-6
    # slot order does not change the result (sum in ascending ROI order)
    perm = [3, 1, 5, 0, 2, 4]
    got2 = cpu(plan.combine(gpu(cores[perm]), perm))
    assert np.array_equal(got, got2)


def test_global_solvers(lt, orc):
    n, na = 48, 24
    nd = nd_for(n)
    ang = synth.angles_for(na)
    shapes = synth.random_shapes(n, 4, 1, np.random.default_rng(2))
    p = synth.analytic_sinogram(shapes, ang, nd).astype(np.float32)
    plan = lt.Plan(n, ang, nd, [[24, 24]], 4, 2, 1)
    got = cpu(plan.global_sirt(gpu(p), 50, 0.0, math.inf))
    ref = orc.global_box(p.astype(np.float64), ang, n, 50, lo=0.0, hi=np.inf)
    assert relerr(got, ref) <= 1e-3
    got = cpu(plan.global_tv(gpu(p), 10, 0.05, 40))
    ref = orc.global_tv(p.astype(np.float64), ang, n, 10, 0.05, 40)
    assert relerr(got, ref) <= 1e-3


def test_full_size_C4_launch_config_sampled(lt, orc):
    """C4 geometry and the full 256-ROI batch bench.py times, n = 3 iterations;
    8 sampled ROIs (corners, edges, interior) against the oracle."""
    cfg = synth.config("C4")
    inp = synth.make_inputs("C4")
    n_iter = 3
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, n_iter)
    plan.filter_bank()
    cores = cpu(plan.tv_solve(gpu(inp.sino), cfg.lam, 20))
    sample = np.array([0, 15, 240, 255, 7, 100, 136, 200])
    ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, inp.centres[sample], cfg.radius,
                       cfg.margin, n_iter, mode="tv", lam=cfg.lam, n_fgp=20)
    for k, g in enumerate(sample):
        q = int(np.nonzero(plan.local_rois == g)[0][0])
        assert relerr(cores[q], ref[k]) <= 1e-3, g


def test_determinism_and_empty(lt):
    inp = synth.make_inputs("C1")
    plan = lt.Plan(64, inp.angles, 91, inp.centres, 12, 8, 10)
    plan.filter_bank()
    a = cpu(plan.sirt_solve(gpu(inp.sino)))
    b = cpu(plan.sirt_solve(gpu(inp.sino)))
    assert np.array_equal(a, b)
    empty = lt.Plan(64, inp.angles, 91, np.zeros((0, 2), np.int32), 12, 8, 10)
    assert empty.R == 0
    empty.filter_bank()
    assert empty.sirt_solve(gpu(inp.sino)).shape == (0, 24, 24)


def test_tv_solve_C2_full(lt, orc):
    """C2 exactly as configured: 512^2, 64 angles, 16 seeded ROIs, TV lambda 0.05,
    200 iterations x 100 FGP iterations, disc on; every ROI core vs the oracle."""
    cfg = synth.config("C2")
    inp = synth.make_inputs("C2")
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, cfg.n_iter)
    plan.filter_bank()
    cores = cpu(plan.tv_solve(gpu(inp.sino), cfg.lam, cfg.n_fgp))
    ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, inp.centres, cfg.radius, cfg.margin,
                       cfg.n_iter, mode="tv", lam=cfg.lam, n_fgp=cfg.n_fgp)
    for q, g in enumerate(plan.local_rois):
        assert relerr(cores[q], ref[g]) <= 1e-3, g
    # combine of the full batch vs the oracle's stitch of the oracle cores
    img = cpu(plan.combine(gpu(cores), plan.local_rois))
    assert relerr(img, orc.stitch(cfg.n, inp.centres, cfg.radius, ref)) <= 1e-3


def test_full_size_C5_sampled(lt, orc):
    """C5 geometry (4096^2, 256 angles, 5793 bins) with the full 1024-ROI batch,
    nonneg SIRT, n = 3; 6 sampled ROIs against the oracle."""
    cfg = synth.config("C5")
    inp = synth.make_inputs("C5")
    n_iter = 3
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, n_iter)
    plan.filter_bank()
    cores = cpu(plan.sirt_solve(gpu(inp.sino), 0.0, math.inf))
    sample = np.array([0, 31, 992, 1023, 500, 529])
    ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, inp.centres[sample], cfg.radius,
                       cfg.margin, n_iter, mode="box")
    for k, g in enumerate(sample):
        q = int(np.nonzero(plan.local_rois == g)[0][0])
        assert relerr(cores[q], ref[k]) <= 1e-3, g


def test_host_buffer_entry_matches_device_path(lt):
    """lt_solve_host (the e2e entry bench.py times) == device solve + combine."""
    cfg = synth.config("C1")
    inp = synth.make_inputs("C1")
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, 20)
    plan.filter_bank()
    cores = plan.sirt_solve(gpu(inp.sino), 0.0, math.inf)
    img_dev = cpu(plan.combine(cores, plan.local_rois))
    img_host = plan.solve_host("sirt", torch.from_numpy(inp.sino).pin_memory(), 0.0, math.inf)
    torch.cuda.synchronize()
    assert np.array_equal(img_host.numpy().astype(np.float64), img_dev)


# ------------------------------------------------------------------ NEXT-3: truncated data

@pytest.mark.parametrize("na,nt,nd", [(512, 257, 1449), (7, 1, 91), (3, 91, 91), (40, 31, 91)])
def test_pad_truncated_exact(lt, orc, na, nt, nd):
    """lt_pad_truncated is a copy: bit-exact against the oracle (T1 size and edge cases)."""
    p = np.random.default_rng(nt).random((na, nt)).astype(np.float32)
    got = cpu(lt.pad_truncated(gpu(p), nd))
    assert np.array_equal(got, orc.pad_truncated(p.astype(np.float64), nd))


def test_pad_truncated_rejects(lt):
    with pytest.raises(ValueError):
        lt.pad_truncated(gpu(np.zeros((4, 9))), 10)      # odd difference
    with pytest.raises(ValueError):
        lt.pad_truncated(gpu(np.zeros((4, 9))), 7)       # target smaller than the data


def test_truncated_tv_solve(lt, orc):
    """T1 recipe at C1 size: central 31 of 91 bins measured, padded on the GPU,
    then the local FISTA-TV path, against the oracle on the oracle's padding."""
    cfg = synth.Config(21, "trunc-small", 64, 48, math.pi, 91, "poisson", 1e4, 1, 12, 8, "centre", 15, "tv",
                       0.05, 40, 5, 0, 31)
    inp = synth.make_inputs(cfg)
    assert inp.sino_trunc.shape == (48, 31)
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, cfg.n_iter)
    plan.filter_bank()
    padded = lt.pad_truncated(gpu(inp.sino_trunc), cfg.n_det)
    cores = cpu(plan.tv_solve(padded, cfg.lam, cfg.n_fgp))
    ref = orc.pipeline(orc.pad_truncated(inp.sino_trunc.astype(np.float64), cfg.n_det), inp.angles, cfg.n,
                       inp.centres, cfg.radius, cfg.margin, cfg.n_iter, mode="tv", lam=cfg.lam, n_fgp=cfg.n_fgp)
    assert relerr(cores[0], ref[0]) <= 1e-3


# ------------------------------------------------------------------ NEXT-4(i): exact x_s

def test_exact_xs_full_grid_is_global_box_sirt(lt, orc):
    """P9 on the GPU: with x_s^k = the global SIRT iterate (LT_XS_EXACT) a ROI
    covering the whole grid reproduces global box-SIRT (split exactness,
    eq. sirtitprior): GPU local vs GPU global and vs the oracle."""
    n, na, nit = 48, 30, 25
    inp = synth.make_inputs("C1", n=n, n_angles=na, n_det=nd_for(n))
    plan = lt.Plan(n, inp.angles, nd_for(n), [[n // 2, n // 2]], n // 2, 0, nit, xs_exact=True)
    core = cpu(plan.sirt_solve(gpu(inp.sino), 0.0, math.inf))[0]
    glob = cpu(plan.global_sirt(gpu(inp.sino), nit, 0.0, math.inf))
    ref = orc.global_box(inp.sino.astype(np.float64), inp.angles, n, nit, lo=0.0, hi=np.inf)
    assert relerr(core, ref) <= 1e-4
    assert relerr(core, glob) <= 1e-4


def test_exact_xs_full_grid_is_global_fista_tv(lt, orc):
    """P10 on the GPU: the same for FISTA-TV (Alg. 3 corrected, A12)."""
    n, na, nit, lam, nf = 32, 24, 10, 0.05, 40
    inp = synth.make_inputs("C1", n=n, n_angles=na, n_det=nd_for(n))
    plan = lt.Plan(n, inp.angles, nd_for(n), [[n // 2, n // 2]], n // 2, 0, nit, xs_exact=True)
    core = cpu(plan.tv_solve(gpu(inp.sino), lam, nf))[0]
    ref = orc.global_tv(inp.sino.astype(np.float64), inp.angles, n, nit, lam, nf)
    assert relerr(core, ref) <= 1e-3


@pytest.mark.parametrize("mode", ["box", "tv"])
def test_exact_xs_local_parity(lt, orc, mode):
    """Exact-x_s local solves on clipped and interior ROIs against the oracle
    fed the oracle's own unconstrained SIRT iterates (xs_exact)."""
    n, na, nit = 64, 32, 12
    inp = synth.make_inputs("C1", n=n, n_angles=na)
    cen = np.array([[32, 32], [12, 50], [52, 14]], dtype=np.int32)
    r, m = 10, 6
    plan = lt.Plan(n, inp.angles, 91, cen, r, m, nit, xs_exact=True)
    p64 = inp.sino.astype(np.float64)
    _, xs = orc.global_box(p64, inp.angles, n, nit, lo=-np.inf, hi=np.inf, iterates=True)
    if mode == "box":
        got = cpu(plan.sirt_solve(gpu(inp.sino), 0.0, math.inf))
        ref = orc.local_solve(n, inp.angles, 91, np.zeros((nit, na, 91)), cen, r, m, mode="box", xs_exact=xs)
    else:
        got = cpu(plan.tv_solve(gpu(inp.sino), 0.05, 30))
        ref = orc.local_solve(n, inp.angles, 91, np.zeros((nit, na, 91)), cen, r, m, mode="tv", lam=0.05,
                              n_fgp=30, xs_exact=xs)
    for q in range(3):
        assert relerr(got[q], ref[q]) <= 1e-3, q


# ------------------------------------------------------------------ NEXT-1: lambda sweep, metrics, Nelder-Mead

@pytest.mark.parametrize("cnt,h,w,rng_L", [(5, 24, 24, None), (3, 64, 48, None), (2, 11, 11, 2.0), (2, 9, 30, None)])
def test_metrics_parity(lt, orc, cnt, h, w, rng_L):
    """lt_metrics (MSE, SSIM) against the oracle's explicit definitions, 1e-6 absolute."""
    g = np.random.default_rng(h * w).random((cnt, h, w)).astype(np.float32)
    x = (g + 0.08 * np.random.default_rng(cnt).standard_normal(g.shape)).astype(np.float32)
    mse, ssim = lt.metrics(gpu(x), gpu(g), rng_L)
    mse, ssim = cpu(mse), cpu(ssim)
    for i in range(cnt):
        assert abs(mse[i] - orc.mse(x[i], g[i])) <= 1e-6 * max(1.0, orc.mse(x[i], g[i]))
        assert abs(ssim[i] - orc.ssim(x[i], g[i], rng_L)) <= 1e-6, (i, ssim[i])
    same = cpu(lt.metrics(gpu(g), gpu(g))[1])
    assert np.all(np.abs(same - (1.0 if h >= 11 and w >= 11 else 0.0)) < 1e-9)


def test_lambda_sweep_matches_per_lambda_solves(lt, orc):
    """One plan holding the same ROI with several lambdas (lt_tv_solve_lambdas)
    equals the oracle's separate solves, and lambda = 0 gives the unregularized path."""
    cfg = synth.Config(22, "sweep", 96, 24, math.pi, 137, "poisson", 1e4, 4, 14, 10, "centre", 8, "tv",
                       0.05, 30, 6, 0)
    inp = synth.make_inputs(cfg)
    lams = [0.0, 0.01, 0.05, 0.3]
    cen = np.repeat(np.array([[48, 40]], dtype=np.int32), len(lams), axis=0)
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, cen, cfg.radius, cfg.margin, cfg.n_iter)
    plan.filter_bank()
    got = cpu(plan.tv_solve(gpu(inp.sino), lams, cfg.n_fgp))
    for q, lam in enumerate(lams):
        ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, cen[:1], cfg.radius, cfg.margin,
                           cfg.n_iter, mode="tv", lam=lam, n_fgp=cfg.n_fgp)
        assert relerr(got[q], ref[0]) <= 1e-3, lam
    single = cpu(plan.tv_solve(gpu(inp.sino), 0.05, cfg.n_fgp))
    assert relerr(got[2], single[2]) <= 1e-6


def test_optimize_lambda(lt, orc):
    """Nelder-Mead over log10(lambda) driving GPU solves + metrics:
    same trajectory as the oracle's Nelder-Mead on the same GPU objective, result
    inside the bounds and no worse than the initial simplex."""
    cfg = synth.Config(23, "tune", 64, 32, math.pi, 91, "poisson", 3e3, 1, 12, 8, "centre", 10, "tv",
                       0.05, 30, 5, 0)
    inp = synth.make_inputs(cfg)
    truth = synth.raster(inp.shapes, cfg.n)
    r0, c0 = 32 - 12, 32 - 12
    ref_core = gpu(truth[r0:r0 + 24, c0:c0 + 24][None])
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, cfg.n_iter)
    plan.filter_bank()
    sino = gpu(inp.sino)
    lam, val, n = plan.optimize_lambda(sino, ref_core, "mse", (-3.0, 0.0), budget=12, n_fgp=cfg.n_fgp)
    assert 1e-3 <= lam <= 1.0 and n <= 12

    def obj(t):
        c = plan.tv_solve(sino, 10.0 ** t, cfg.n_fgp)
        return float(lt.metrics(c, ref_core)[0].mean())
    t_ref, v_ref, n_ref = orc.nelder_mead_1d(obj, -3.0, 0.0, 12)
    assert abs(math.log10(lam) - t_ref) < 1e-12 and n == n_ref and abs(val - v_ref) <= 1e-9 * max(v_ref, 1e-30)
    assert val <= min(obj(-1.5), obj(-1.0)) + 1e-12
    lam_s, val_s, _ = plan.optimize_lambda(sino, ref_core, "ssim", (-3.0, 0.0), budget=8, n_fgp=cfg.n_fgp)
    assert 1e-3 <= lam_s <= 1.0 and 0.0 < val_s <= 1.0


# ------------------------------------------------------------------ NEXT-2: Haar l1 prior

@pytest.mark.parametrize("momentum,levels", [(True, 4), (False, 3), (True, 0)])
def test_haar_solve_parity(lt, orc, momentum, levels):
    """Local Haar-l1 reconstruction (FISTA / ISTA) against the oracle, clipped and
    interior ROIs whose extended sides are divisible by 2^levels."""
    cfg = synth.Config(24, "haar", 96, 30, math.pi, 137, "poisson", 1e4, 3, 16, 16, "seeded", 10, "tv",
                       0.05, 30, 6, 0)
    inp = synth.make_inputs(cfg)
    cen = np.array([[48, 48], [16, 64], [80, 32]], dtype=np.int32)   # extended sides 64, 48x64, 48x64
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, cen, cfg.radius, cfg.margin, cfg.n_iter)
    plan.filter_bank()
    lam = 0.02
    got = cpu(plan.haar_solve(gpu(inp.sino), lam, levels, momentum))
    ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, cen, cfg.radius, cfg.margin, cfg.n_iter,
                       mode="haar", lam=lam, levels=levels) if momentum else None
    if not momentum:
        pc, c, _, _ = orc.disc(inp.sino.astype(np.float64), inp.angles, cfg.n)
        b = orc.conv_cache(orc.filter_bank(cfg.n, inp.angles, cfg.n_det, cfg.n_iter), pc)
        ref = orc.local_solve(cfg.n, inp.angles, cfg.n_det, b, cen, cfg.radius, cfg.margin, mode="haar", lam=lam,
                              levels=levels, momentum=False, disc_c=c, use_disc=True)
    for q in range(3):
        assert relerr(got[q], ref[q]) <= 1e-3, q


def test_haar_solve_rejects_indivisible(lt):
    inp = synth.make_inputs("C1")
    plan = lt.Plan(64, inp.angles, 91, [[30, 30]], 12, 8, 5)      # extended side 40: not divisible by 16
    plan.filter_bank()
    with pytest.raises(ValueError):
        plan.haar_solve(gpu(inp.sino), 0.01, 4)
    plan.haar_solve(gpu(inp.sino), 0.01, 3)                      # 40 = 5 * 8


# ------------------------------------------------------------------ NEXT-4(iii): Chambolle-Pock TV

@pytest.mark.parametrize("n,na,mu_scale", [(64, 32, 0.05), (48, 24, 0.0)])
def test_global_cp_parity(lt, orc, n, na, mu_scale):
    """Preconditioned Chambolle-Pock on the full grid against the oracle, same
    iteration count (the iteration map is the same; fp32 vs fp64 only)."""
    nd = nd_for(n)
    inp = synth.make_inputs("C1", n=n, n_angles=na, n_det=nd)
    mu = mu_scale * na * nd                     # mu = lambda / alpha
    plan = lt.Plan(n, inp.angles, nd, [[n // 2, n // 2]], 8, 4, 2)
    got = cpu(plan.global_cp(gpu(inp.sino), 40, mu))
    ref = orc.global_cp(inp.sino.astype(np.float64), inp.angles, n, 40, mu)
    assert relerr(got, ref) <= 1e-3


# ------------------------------------------------------------------ NEXT-4(ii): exterior subtraction

def test_exterior_solve_parity(lt, orc):
    """Exterior subtraction (prior art) with xg = FBP with the SIRT
    filter u_n + c D: GPU against the oracle on interior and clipped ROIs."""
    cfg = synth.config("C1")
    inp = synth.make_inputs(cfg)
    cen = np.array([[32, 32], [12, 50], [50, 14]], dtype=np.int32)
    nit = 15
    plan = lt.Plan(64, inp.angles, 91, cen, 12, 8, nit)
    plan.filter_bank()
    got = cpu(plan.exterior_solve(gpu(inp.sino), 0.0, math.inf))
    p64 = inp.sino.astype(np.float64)
    xg = orc.fbp_filtered(p64, inp.angles, 64, nit)
    ref = orc.exterior_solve(p64, inp.angles, 64, xg, cen, 12, 8, nit)
    for q in range(3):
        assert relerr(got[q], ref[q]) <= 1e-3, q


def test_exterior_solve_full_grid_is_global_sirt(lt, orc):
    """Full-grid ROI: no exterior, so the result is global box-SIRT (GPU vs GPU and oracle)."""
    inp = synth.make_inputs("C1", n=48, n_angles=24, n_det=nd_for(48))
    nit = 12
    plan = lt.Plan(48, inp.angles, nd_for(48), [[24, 24]], 24, 0, nit)
    plan.filter_bank()
    core = cpu(plan.exterior_solve(gpu(inp.sino), 0.0, math.inf))[0]
    ref = orc.global_box(inp.sino.astype(np.float64), inp.angles, 48, nit)
    assert relerr(core, ref) <= 1e-4


def test_tv_solve_C3_subset(lt, orc):
    """C3 geometry (limited angle, extended side 192: 6-CTA FGP clusters) with the
    TV solver on seeded (partly clipped) ROIs, 12 iterations x 30 FGP steps."""
    cfg = synth.config("C3")
    inp = synth.make_inputs("C3")
    n_iter, n_fgp = 12, 30
    cen = np.concatenate([inp.centres[:3], np.array([[48, 48], [976, 960]], dtype=np.int32)])
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, cen, cfg.radius, cfg.margin, n_iter)
    plan.filter_bank()
    cores = cpu(plan.tv_solve(gpu(inp.sino), cfg.lam, n_fgp))
    ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, cen, cfg.radius, cfg.margin, n_iter,
                       mode="tv", lam=cfg.lam, n_fgp=n_fgp)
    for q in range(len(cen)):
        assert relerr(cores[q], ref[q]) <= 1e-3, q


_GRAPH_SCRIPT = r"""
import sys, math, numpy as np, torch
sys.path.insert(0, '.')
import synth, paper_1604_02292_b200 as lt
cfg = synth.config("C1"); inp = synth.make_inputs("C1")
plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, cfg.n_iter)
plan.filter_bank()
outs = []
for k in range(3):                      # capture, then replays with new data
    sino = torch.from_numpy(inp.sino * (1.0 + 0.1 * k)).float().cuda()
    outs.append(plan.sirt_solve(sino, 0.0, math.inf).cpu().numpy())
    outs.append(plan.tv_solve(sino, 0.05, 30).cpu().numpy())
np.save(sys.argv[1], np.stack(outs))
"""


def test_graph_replay_matches_eager(lt, tmp_path):
    """The CUDA-graph replay of the local iteration loop (forced on) gives the
    same bits as eager launches (forced off), including replays with new data."""
    import subprocess, sys as _sys
    res = {}
    for g in ("0", "1"):
        f = tmp_path / f"g{g}.npy"
        env = dict(os.environ, LT_GRAPH=g)
        r = subprocess.run([_sys.executable, "-c", _GRAPH_SCRIPT, str(f)], env=env, capture_output=True, text=True,
                           cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res[g] = np.load(f)
    assert np.array_equal(res["0"], res["1"])


@pytest.mark.parametrize("n_iter,radius,margin", [(1, 8, 4), (2, 1, 0), (3, 1, 3), (1, 31, 0)])
def test_degenerate_solves(lt, orc, n_iter, radius, margin):
    """Edge cases of the method: one outer iteration (x_s^1 only, y^0 = 0), a
    2x2 core with no margin, a margin wider than the core, a core touching the
    grid edge; box-SIRT and FISTA-TV against the oracle."""
    cfg = synth.Config(23, "degenerate", 64, 20, math.pi, 91, "gauss", 0.01, 1, radius, margin, "centre", n_iter,
                       "tv", 0.05, 10, 3, 0)
    inp = synth.make_inputs(cfg)
    cen = np.array([[32, 32], [radius, 64 - radius]], dtype=np.int32)
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, cen, radius, margin, n_iter)
    plan.filter_bank()
    sino = gpu(inp.sino)
    box = cpu(plan.sirt_solve(sino, 0.0, math.inf))
    tv = cpu(plan.tv_solve(sino, cfg.lam, cfg.n_fgp))
    ref_box = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, cen, radius, margin, n_iter, mode="box")
    ref_tv = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, cen, radius, margin, n_iter, mode="tv",
                          lam=cfg.lam, n_fgp=cfg.n_fgp)
    for q in range(len(cen)):
        assert relerr(box[q], ref_box[q]) <= 1e-3, ("box", q)
        assert relerr(tv[q], ref_tv[q]) <= 1e-3, ("tv", q)


def test_determinism_full_size_c4(lt):
    """Bitwise-identical repeated solves in bench.py's C4 launch configuration
    (24-angle projector CTAs, 64x64 backprojection blocks, 8-CTA FGP clusters,
    the side-stream x_s backprojection with its events), TV and box."""
    cfg = synth.config("C4")
    inp = synth.make_inputs("C4")
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, 4)
    plan.filter_bank()
    sino = gpu(inp.sino)
    tv = [cpu(plan.tv_solve(sino, cfg.lam, 10)) for _ in range(3)]
    box = [cpu(plan.sirt_solve(sino, 0.0, math.inf)) for _ in range(2)]
    assert np.array_equal(tv[0], tv[1]) and np.array_equal(tv[0], tv[2])
    assert np.array_equal(box[0], box[1])


def test_two_group_pipelining_matches_oracle(lt, orc, monkeypatch):
    """LT_SPLIT=2 (two ROI groups on their own streams, one shared side-stream
    x_s^k, the second group of LT_SPLIT_B ROIs): C2's 16 ROIs as 13 + 3, TV and
    box, against the oracle and against the one-group solve."""
    cfg = synth.config("C2")
    inp = synth.make_inputs("C2")
    n_iter = 12
    sino = gpu(inp.sino)
    base = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, n_iter)
    base.filter_bank()
    bank = base.get_bank()
    want_tv = cpu(base.tv_solve(sino, cfg.lam, 30))
    want_box = cpu(base.sirt_solve(sino, 0.0, math.inf))
    monkeypatch.setenv("LT_SPLIT", "2")
    monkeypatch.setenv("LT_SPLIT_B", "3")
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, n_iter)
    plan.set_bank(bank)
    got_tv = cpu(plan.tv_solve(sino, cfg.lam, 30))
    got_box = cpu(plan.sirt_solve(sino, 0.0, math.inf))
    assert relerr(got_tv, want_tv) <= 1e-5 and relerr(got_box, want_box) <= 1e-5
    sample = np.array([0, 5, 13, 15])          # both groups
    ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, inp.centres[sample], cfg.radius,
                       cfg.margin, n_iter, mode="tv", lam=cfg.lam, n_fgp=30)
    for k, g in enumerate(sample):
        q = int(np.nonzero(plan.local_rois == g)[0][0])
        assert relerr(got_tv[q], ref[k]) <= 1e-3, g
