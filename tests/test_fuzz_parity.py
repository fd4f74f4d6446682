"""Seeded random geometries against the fp64 oracle (GPU): grid sizes, angle
counts and spans, detector counts, ROI radii / margins / positions (clipped or
not, overlapping or not), iteration counts and priors drawn at random, so the
launch-shape decisions (split launches, FGP cluster shapes, small-batch
backprojection, tile widths) are exercised on shapes no config names."""
import math
import os

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
    return m


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


def relerr(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(24, 321))
    na = int(rng.integers(3, 97))
    span = math.pi if rng.random() < 0.7 else 2 * math.pi / 3
    nd = int(math.ceil(math.sqrt(2) * n)) | 1
    nd += 2 * int(rng.integers(0, 3))                       # wider detectors too (odd N_d)
    radius = int(rng.integers(1, max(2, n // 4)))
    margin = int(rng.integers(0, 33))
    n_roi = int(rng.integers(1, 6))
    cen = np.stack([rng.integers(radius, n - radius + 1, size=n_roi),
                    rng.integers(radius, n - radius + 1, size=n_roi)], axis=1).astype(np.int32)
    n_iter = int(rng.integers(1, 6))
    mode = "tv" if rng.random() < 0.5 else "box"
    cfg = synth.Config(40 + seed, f"fuzz{seed}", n, na, span, nd, "gauss", 0.01, n_roi, radius, margin, "seeded",
                       n_iter, mode, 0.05, int(rng.integers(5, 31)), 4, 0)
    return cfg, cen


# LT_FUZZ_SEEDS widens the sweep for one-off stress runs (profiles/r01/fuzz_*.txt)
@pytest.mark.parametrize("seed", range(int(os.environ.get("LT_FUZZ_SEEDS", "40"))))
def test_random_geometry(lt, orc, seed):
    cfg, cen = _case(seed)
    inp = synth.make_inputs(cfg)
    h = cfg.radius + cfg.margin
    if 2 * h > 320 and cfg.solver == "tv":
        pytest.skip("FGP tiles are limited to 320 x 320")
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, cen, cfg.radius, cfg.margin, cfg.n_iter)
    plan.filter_bank()
    sino = torch.from_numpy(inp.sino).cuda()
    if cfg.solver == "tv":
        got = plan.tv_solve(sino, cfg.lam, cfg.n_fgp).cpu().numpy()
        ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, cen, cfg.radius, cfg.margin, cfg.n_iter,
                           mode="tv", lam=cfg.lam, n_fgp=cfg.n_fgp)
    else:
        got = plan.sirt_solve(sino, 0.0, math.inf).cpu().numpy()
        ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, cen, cfg.radius, cfg.margin, cfg.n_iter,
                           mode="box")
    for q in range(len(cen)):
        assert relerr(got[q], ref[q]) <= 1e-3, (cfg, q)


@pytest.mark.parametrize("seed", range(6))
def test_random_geometry_large_batch(lt, orc, seed):
    """Many ROIs (60-300) on random geometries: the large-batch launch shapes
    (16 angles per FP CTA, 64x64 backprojection blocks, 8-CTA FGP clusters)
    on 8 sampled ROIs against the oracle."""
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.integers(200, 513))
    na = int(rng.integers(60, 181))
    nd = int(math.ceil(math.sqrt(2) * n)) | 1
    radius = int(rng.integers(8, 41))
    margin = int(rng.integers(0, 49))
    n_roi = int(rng.integers(60, 301))
    cen = np.stack([rng.integers(radius, n - radius + 1, size=n_roi),
                    rng.integers(radius, n - radius + 1, size=n_roi)], axis=1).astype(np.int32)
    mode = "tv" if seed % 2 == 0 else "box"
    cfg = synth.Config(80 + seed, f"fuzzL{seed}", n, na, math.pi, nd, "gauss", 0.01, n_roi, radius, margin, "seeded",
                       int(rng.integers(1, 4)), mode, 0.05, 15, 6, 0)
    inp = synth.make_inputs(cfg)
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, cen, cfg.radius, cfg.margin, cfg.n_iter)
    plan.filter_bank()
    sino = torch.from_numpy(inp.sino).cuda()
    got = (plan.tv_solve(sino, cfg.lam, cfg.n_fgp) if mode == "tv" else plan.sirt_solve(sino, 0.0, math.inf)).cpu().numpy()
    sample = np.unique(np.concatenate([[0, n_roi - 1], rng.integers(0, n_roi, size=6)]))
    ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, cen[sample], cfg.radius, cfg.margin, cfg.n_iter,
                       mode=mode, lam=cfg.lam, n_fgp=cfg.n_fgp)
    for k, g in enumerate(sample):
        q = int(np.nonzero(plan.local_rois == g)[0][0])
        assert relerr(got[q], ref[k]) <= 1e-3, (cfg, int(g))


@pytest.mark.parametrize("seed", range(int(os.environ.get("LT_FUZZ_WIDE", "8"))))
def test_random_geometry_wide_tiles(lt, orc, seed):
    """Extended sides of 258..320 px (the 10-columns-per-lane FGP, the wide
    forward projector), central and clipped ROIs, box or TV, on random
    geometries against the oracle."""
    rng = np.random.default_rng(3000 + seed)
    n = int(rng.integers(300, 641))
    na = int(rng.integers(16, 97))
    nd = int(math.ceil(math.sqrt(2) * n)) | 1
    side = int(rng.integers(129, 161))                      # extended half-side h in (128, 160]
    radius = int(rng.integers(max(1, side - 64), min(side, n // 2) + 1))
    margin = side - radius
    n_roi = int(rng.integers(1, 4))
    cen = np.stack([rng.integers(radius, n - radius + 1, size=n_roi),
                    rng.integers(radius, n - radius + 1, size=n_roi)], axis=1).astype(np.int32)
    mode = "tv" if seed % 2 == 0 else "box"
    cfg = synth.Config(90 + seed, f"fuzzW{seed}", n, na, math.pi, nd, "gauss", 0.01, n_roi, radius, margin, "seeded",
                       int(rng.integers(1, 4)), mode, 0.05, int(rng.integers(5, 21)), 6, 2)
    inp = synth.make_inputs(cfg)
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, cen, cfg.radius, cfg.margin, cfg.n_iter)
    assert 2 * plan.h > 256
    plan.filter_bank()
    sino = torch.from_numpy(inp.sino).cuda()
    got = (plan.tv_solve(sino, cfg.lam, cfg.n_fgp) if mode == "tv" else plan.sirt_solve(sino, 0.0, math.inf)).cpu().numpy()
    ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, cen, cfg.radius, cfg.margin, cfg.n_iter,
                       mode=mode, lam=cfg.lam, n_fgp=cfg.n_fgp)
    for q, g in enumerate(plan.local_rois):
        assert relerr(got[q], ref[g]) <= 1e-3, (cfg, int(g))
