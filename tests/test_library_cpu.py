"""Host-side checks of the C-ABI library (-m "not gpu"): it loads, exports every
symbol include/loctomo.h declares, validates arguments (error code 2), and
its ROI plan (rectangles, windows, partition) is exact against the oracle and
brute force.  No device compute is called here."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lt():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1604_02292_b200 as m
    return m


def header_symbols():
    src = open(os.path.join(ROOT, "include", "loctomo.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lt_\w+)\s*\(", src)))


def test_exports_every_header_symbol(lt):
    lib = ctypes.CDLL(lt.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(lt.EXPORTS)


def _setup(lt, n=64, angles=None, nd=91, cen=((32, 32),), r=12, m=8, nit=10, rank=0, world=1):
    angles = synth.angles_for(32) if angles is None else np.asarray(angles, dtype=np.float64)
    cen = np.asarray(cen, dtype=np.int32).reshape(-1, 2)
    rows = np.ascontiguousarray(cen[:, 0]); cols = np.ascontiguousarray(cen[:, 1])
    p = ctypes.c_void_p()
    rc = lt._lib.lt_roi_setup(n, len(angles), nd, angles.ctypes.data, len(cen), rows.ctypes.data, cols.ctypes.data,
                              r, m, nit, 1, rank, world, ctypes.byref(p))
    if rc == 0:
        lt._lib.lt_plan_destroy(p)
    return rc


def test_argument_validation(lt):
    assert _setup(lt) == 0
    assert _setup(lt, nd=90) == 2                                   # even N_d
    assert _setup(lt, angles=[0.0, 0.5, 0.4]) == 2                  # not increasing
    assert _setup(lt, angles=[0.0, 3.2]) == 2                       # outside [0, pi)
    assert _setup(lt, cen=((5, 32),)) == 2                          # core outside the grid
    assert _setup(lt, r=0) == 2
    assert _setup(lt, m=-1) == 2
    assert _setup(lt, nit=0) == 2
    assert _setup(lt, rank=2, world=2) == 2
    assert _setup(lt, n=0) == 2
    assert _setup(lt, cen=np.zeros((0, 2))) == 0                    # empty ROI list is valid


def test_unbound_plan_errors(lt):
    plan = lt.Plan(64, synth.angles_for(8), 91, [[32, 32]], 12, 8, 5, bind=False)
    rc = lt._lib.lt_filter_bank(plan._p, None)
    assert rc == 2 and b"workspace" in lt._lib.lt_last_error()


def test_rects_match_oracle(lt, orc):
    for cfg in ("C1", "C2", "C3", "C4"):
        c = synth.config(cfg)
        cen = synth.roi_centres(c)
        plan = lt.Plan(c.n, synth.angles_for(c.n_angles, c.span), c.n_det, cen, c.radius, c.margin, 1, bind=False)
        rects, _, _ = plan.tables()
        ref = orc.roi_rects(c.n, cen, c.radius, c.margin)
        h = c.radius + c.margin
        for q, g in enumerate(plan.local_rois):
            row0, col0, vr0, vr1, vc0, vc1 = rects[q]
            assert (row0 + vr0, row0 + vr1, col0 + vc0, col0 + vc1) == tuple(ref[g][4:8])
            assert (row0 + h - c.radius, col0 + h - c.radius) == (ref[g][0], ref[g][2])


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_windows_contain_exact_support(lt, orc, cfg):
    """P12: each ROI's window [d0, d0 + W) contains every bin where W_{L'} is
    nonzero (brute force with the oracle's W on the indicator of L')."""
    c = synth.config(cfg)
    ang = synth.angles_for(c.n_angles, c.span)
    cen = np.concatenate([synth.roi_centres(c)[:4], [[c.radius, c.radius], [c.n - c.radius, c.n - c.radius]]])
    plan = lt.Plan(c.n, ang, c.n_det, cen, c.radius, c.margin, 1, bind=False)
    rects, d0, W = plan.tables()
    assert W == lt.window_width(c.radius + c.margin)
    ref = orc.roi_rects(c.n, cen, c.radius, c.margin)
    ones = np.ones((c.n, c.n))
    for q, g in enumerate(plan.local_rois):
        s = orc.forward(ones, ang, c.n_det, tuple(int(v) for v in ref[g][4:8]))
        for a in range(c.n_angles):
            nz = np.nonzero(s[a])[0]
            assert nz.min() >= d0[q, a] and nz.max() < d0[q, a] + W, (cfg, g, a)


def test_window_width_bruteforce():
    """W(h) = 2 ceil((2h-1)/sqrt2) + 4 >= the support width of a 2h x 2h square
    at any angle and any sub-bin offset of its centre (V4)."""
    import paper_1604_02292_b200 as m
    rng = np.random.default_rng(0)
    for h in (1, 2, 5, 20, 64, 96, 128):
        W = m.window_width(h)
        for _ in range(400):
            th = rng.uniform(0, math.pi)
            c = max(abs(math.cos(th)), abs(math.sin(th)))
            tau = rng.uniform(-50, 50)
            half = (h - 0.5) * (abs(math.cos(th)) + abs(math.sin(th)))
            lo = math.floor(tau - half - c) + 1          # smallest bin strictly inside the support
            hi = math.ceil(tau + half + c) - 1
            d0 = math.floor(tau) - W // 2
            assert lo >= d0 and hi < d0 + W, (h, th, tau)


@pytest.mark.parametrize("cfg_name", ["C2", "C4", "C5"])
def test_partition_covers_every_roi_once(lt, cfg_name):
    """Contiguous raster-order partition: every ROI on exactly one rank, local
    lists ascending, cost balanced within one ROI's cost, ranks spatially compact
    (for the C4/C5 tilings each rank's cores span at most ceil(rows/world) + 1 tile rows)."""
    c = synth.config(cfg_name)
    cen = synth.roi_centres(c)
    ang = synth.angles_for(8)
    h = c.radius + c.margin
    def cost(r):
        hv = min(c.n, cen[r, 0] + h) - max(0, cen[r, 0] - h)
        wv = min(c.n, cen[r, 1] + h) - max(0, cen[r, 1] - h)
        return 4 * (2 * h) ** 2 + 3 * hv * wv
    for world in (1, 2, 3, 4, 8):
        seen, loads = [], []
        for rank in range(world):
            plan = lt.Plan(c.n, ang, c.n_det, cen, c.radius, c.margin, 1, rank=rank, world=world, bind=False)
            assert np.all(np.diff(plan.local_rois) > 0)
            seen.extend(plan.local_rois.tolist())
            loads.append(sum(cost(r) for r in plan.local_rois))
            if c.layout == "tiling" and plan.R:
                rows = np.unique(cen[plan.local_rois, 0])
                assert len(rows) <= -(-(c.n // (2 * c.radius)) // world) + 1
        assert sorted(seen) == list(range(len(cen)))
        assert max(loads) - sum(loads) / world <= max(cost(r) for r in range(len(cen)))


def test_workspace_size_reasonable(lt):
    c = synth.config("C5")
    plan = lt.Plan(c.n, synth.angles_for(c.n_angles), c.n_det, synth.roi_centres(c), c.radius, c.margin,
                   c.n_iter, bind=False)
    gb = plan.workspace_bytes / 2**30
    assert 5.0 < gb < 40.0, gb          # bank + conv cache (2 x 2.97 GB) + ROI state fit 180 GB


@pytest.mark.parametrize("fn,lo,hi,budget", [
    (lambda t: (t - 2.0) ** 2, -3.0, 4.0, 50),
    (lambda t: (t - 2.0) ** 2, -3.0, 4.0, 3),
    (lambda t: t, -3.0, 4.0, 40),
    (lambda t: abs(math.sin(3.0 * t)) + 0.1 * t * t, -2.0, 1.0, 25),
])
def test_nelder_mead_matches_oracle(lt, orc, fn, lo, hi, budget):
    """lt_nelder_mead_1d (host code of the library, NEXT-1) follows the same
    deterministic trajectory as the oracle's independent implementation."""
    a, b = [], []
    got = lt.nelder_mead_1d(lambda t: a.append(t) or fn(t), lo, hi, budget)
    ref = orc.nelder_mead_1d(lambda t: b.append(t) or fn(t), lo, hi, budget)
    assert got == ref and a == b


def test_nelder_mead_validation(lt):
    with pytest.raises(ValueError):
        lt.nelder_mead_1d(lambda t: t, 1.0, 1.0, 10)
    with pytest.raises(ValueError):
        lt.nelder_mead_1d(lambda t: t, 0.0, 1.0, 2)


def test_bank_key_depends_on_geometry_only(lt):
    """lt_bank_key: what Alg. 1's filters depend on (N, angles, N_d, alpha;
    P:L489-503) changes the key; n_iter, the ROI list, radius and margin do not
    (u_k does not depend on n or on the ROIs)."""
    ang = synth.angles_for(16)
    key = lambda **kw: lt.Plan(kw.get("n", 64), kw.get("ang", ang), kw.get("nd", 91), kw.get("cen", [[32, 32]]),
                               kw.get("r", 12), kw.get("m", 8), kw.get("nit", 5), bind=False).bank_key
    k0 = key()
    assert k0 != 0
    assert key(nit=50) == k0 and key(cen=[[20, 20], [40, 40]], r=8, m=2) == k0
    assert key(n=65) != k0 and key(nd=93) != k0 and key(ang=synth.angles_for(17)) != k0
    a2 = ang.copy(); a2[3] = np.nextafter(a2[3], 10.0)
    assert key(ang=a2) != k0


def test_unbound_plan_rejects_bank_calls(lt):
    plan = lt.Plan(64, synth.angles_for(8), 91, [[32, 32]], 12, 8, 5, bind=False)
    assert lt._lib.lt_set_bank(plan._p, None, plan.bank_key, None) == 2
    assert lt._lib.lt_save_bank(plan._p, b"/tmp/x.bank", None) == 2
    assert lt._lib.lt_load_bank(plan._p, b"/tmp/x.bank", None) == 2
    assert lt._lib.lt_combine_rois(plan._p, None, None, None, None) == 2
    assert lt.window_width(64) == 184 and lt.window_width(1) == 6        # 2 ceil((2h-1)/sqrt2) + 4
    assert lt._lib.lt_window_width(0) == -1


def test_output_buffer_checks_host_side():
    import paper_1604_02292_b200 as m
    import torch
    with pytest.raises(TypeError):
        m._out_f32(torch.empty(2, 2), (2, 2), torch.device("cuda", 0))     # host tensor
    with pytest.raises(TypeError):
        m._cuda_f32(torch.empty(2, 2, dtype=torch.float64), "x")


@pytest.mark.parametrize("world", [2, 3, 8])
def test_library_slot_table_matches_partition(lt, world):
    """lt_plan_slot_table = the per-rank local lists of the partition, padded to
    the largest count (the layout lt_combine_rois all-gathers)."""
    c = synth.config("C4")
    cen = synth.roi_centres(c)
    ang = synth.angles_for(c.n_angles, c.span)
    plans = [lt.Plan(c.n, ang, c.n_det, cen, c.radius, c.margin, 1, rank=g, world=world, bind=False)
             for g in range(world)]
    spr = max(p.R for p in plans)
    for p in plans:
        s, tab = p.slot_table()
        assert s == spr and tab.shape == (world * spr,)
        for g, q in enumerate(plans):
            blk = tab[g * spr:(g + 1) * spr]
            assert np.array_equal(blk[:q.R], q.local_rois) and np.all(blk[q.R:] == -1)


def test_tv_accepts_extended_sides_up_to_320(lt):
    """The FGP kernels take extended ROIs up to 320 x 320 (the paper's 256^2 local
    parts with 1/8 padding per side); wider is error 2 (host check)."""
    ang = synth.angles_for(8)
    ok = lt.Plan(1024, ang, 1449, [[512, 512]], 128, 32, 2, bind=False)
    assert ok.h == 160
    assert lt._lib.lt_fgp_batch(320, 320, 0, None, 0.1, 10, None, None) == 0
    assert lt._lib.lt_fgp_batch(321, 320, 1, None, 0.1, 10, None, None) == 2
    assert lt._lib.lt_fgp_batch(300, 321, 1, None, 0.1, 10, None, None) == 2
