"""Pins of the fp64 oracle against things other than itself (-m "not gpu").

Each test names the pin ID of DESIGN.md §Oracle pins and the PAPER.md passage
("P:Lnnn") it fixes.  Plausible mistakes (dropped 1/c factor, wrong sign of
y, transposed index, wrong alpha, half-width-1 backprojector, dropped momentum
term, wrong FGP step) each fail at least one of them.
"""
import math
import os

import numpy as np
import pytest

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def relerr(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def dense_W(orc, n, ang, nd):
    """Matrix of the oracle's forward operator, column by column."""
    W = np.zeros((len(ang) * nd, n * n))
    for k in range(n * n):
        e = np.zeros(n * n); e[k] = 1.0
        W[:, k] = orc.forward(e.reshape(n, n), ang, nd).ravel()
    return W


def joseph_ray_march(img, ang, nd):
    """Independent explicit Joseph projector: for each ray march the rows
    (|cos| >= |sin|) or columns, interpolate linearly between the two
    neighbouring pixel centres, scale by the step length 1/c (V2)."""
    n = img.shape[0]
    h = (n - 1) / 2.0
    out = np.zeros((len(ang), nd))
    for a, th in enumerate(ang):
        c, s = math.cos(th), math.sin(th)
        for d in range(nd):
            t = d - (nd - 1) / 2.0
            acc = 0.0
            if abs(c) >= abs(s):
                for i in range(n):
                    y = h - i
                    x = (t - y * s) / c
                    u = x + h                      # fractional column index
                    j0 = math.floor(u); f = u - j0
                    if 0 <= j0 < n: acc += (1 - f) * img[i, j0]
                    if 0 <= j0 + 1 < n: acc += f * img[i, j0 + 1]
                out[a, d] = acc / abs(c)
            else:
                for j in range(n):
                    x = j - h
                    y = (t - x * c) / s
                    v = h - y                      # fractional row index
                    i0 = math.floor(v); f = v - i0
                    if 0 <= i0 < n: acc += (1 - f) * img[i0, j]
                    if 0 <= i0 + 1 < n: acc += f * img[i0 + 1, j]
                out[a, d] = acc / abs(s)
    return out


# ---------------------------------------------------------------- projector

def test_golden_2x2_closed_form_chords(orc):
    """Hand-derived line integrals on a 2x2 grid (tests/golden/joseph_2x2.txt)."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "joseph_2x2.txt")) if l.strip() and not l.startswith("#")]
    ang = np.array([0.0, math.pi / 4, math.pi / 2, 3 * math.pi / 4])
    Wg = np.zeros((4 * 3, 4))
    for r in rows:
        a, d = int(r[0]), int(r[1])
        Wg[a * 3 + d] = [float(v) for v in r[2:]]
    W = dense_W(orc, 2, ang, 3)
    assert np.max(np.abs(W - Wg)) < 1e-14


@pytest.mark.parametrize("n,nd", [(8, 13), (16, 23), (9, 13)])
def test_P1_closed_form_equals_joseph_ray_march(orc, n, nd):
    """P1: the oracle's closed-form W equals explicit Joseph ray marching (brute force)."""
    ang = np.concatenate([synth.angles_for(12), [math.pi / 4 + 1e-3, 3 * math.pi / 4 - 1e-3, 1.0]])  # includes exact 45/135 deg ties
    ang = np.sort(ang)
    rng = np.random.default_rng(n)
    for _ in range(3):
        x = rng.standard_normal((n, n))
        a = orc.forward(x, ang, nd)
        b = joseph_ray_march(x, ang, nd)
        assert relerr(a, b) < 1e-12


@pytest.mark.parametrize("n", [8, 16, 32, 64])
def test_P2_adjoint_identity(orc, n):
    """P2: <W x, y> = <x, W^T y> to 1e-12 relative (north star)."""
    nd = int(math.ceil(math.sqrt(2) * n)) | 1
    ang = synth.angles_for(2 * n if n < 64 else 40)
    rng = np.random.default_rng(100 + n)
    for _ in range(3):
        x = rng.standard_normal((n, n)); y = rng.standard_normal((len(ang), nd))
        lhs = float(np.vdot(orc.forward(x, ang, nd), y))
        rhs = float(np.vdot(x, orc.back(y, ang, n)))
        assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(x) * np.linalg.norm(y) * math.sqrt(n)
        assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0) * 10


def test_P2_dense_transpose(orc):
    n, nd = 8, 13
    ang = synth.angles_for(10)
    W = dense_W(orc, n, ang, nd)
    WT = np.zeros((n * n, len(ang) * nd))
    for k in range(len(ang) * nd):
        e = np.zeros(len(ang) * nd); e[k] = 1.0
        WT[:, k] = orc.back(e.reshape(len(ang), nd), ang, n).ravel()
    assert np.max(np.abs(WT - W.T)) < 1e-13


def test_P3_axis_closed_forms(orc):
    """P3: theta = 0 -> (Wx)(d) = (colsum(j) + colsum(j+1))/2 with x_j = t_d - 1/2;
    theta = pi/2 -> the same with rows (even N, odd N_d)."""
    n, nd = 10, 15
    x = np.random.default_rng(3).standard_normal((n, n))
    s = orc.forward(x, np.array([0.0, math.pi / 2]), nd)
    col = x.sum(axis=0); row = x.sum(axis=1)
    exp0 = np.zeros(nd); exp90 = np.zeros(nd)
    for d in range(nd):
        t = d - (nd - 1) / 2
        j = int(round(t - 0.5 + (n - 1) / 2))          # x_j = t - 1/2
        exp0[d] = 0.5 * ((col[j] if 0 <= j < n else 0) + (col[j + 1] if 0 <= j + 1 < n else 0))
        i = int(round((n - 1) / 2 - (t + 0.5)))        # y_i = t + 1/2
        exp90[d] = 0.5 * ((row[i] if 0 <= i < n else 0) + (row[i + 1] if 0 <= i + 1 < n else 0))
    assert np.max(np.abs(s[0] - exp0)) < 1e-13
    assert np.max(np.abs(s[1] - exp90)) < 1e-12


def test_P4_analytic_chord_lengths_converge(orc):
    """P4: W applied to an 8x supersampled raster of a disc / ellipse approaches
    the analytic line integrals at rate ~1/N (closed form within the discretization bound)."""
    errs = {}
    for n in (128, 256, 512):
        nd = int(math.ceil(math.sqrt(2) * n)) | 1
        ang = synth.angles_for(16)
        shapes = {"disc": [synth.Shape("ellipse", 0.05 * n, -0.1 * n, 0.3 * n, 0.3 * n, 0.0, 1.0)],
                  "ellipse": [synth.Shape("ellipse", -0.07 * n, 0.03 * n, 0.33 * n, 0.18 * n, 0.6, 1.0)]}
        for name, sh in shapes.items():
            img = synth.raster(sh, n, supersample=8)
            p_num = orc.forward(img, ang, nd)
            p_ana = synth.analytic_sinogram(sh, ang, nd, subrays=(0.0,))
            errs[(name, n)] = relerr(p_num, p_ana)
    for name in ("disc", "ellipse"):
        for n in (128, 256, 512):
            assert errs[(name, n)] <= 2.0 / n, (name, n, errs[(name, n)])
        ratio = errs[(name, 128)] / errs[(name, 512)]     # first order: 4 per two doublings
        assert 3.0 <= ratio <= 5.3, (name, ratio)


def test_P12_masks_and_split(orc):
    """P12: W_L x = W(M_L x), W_L^T = M_L W^T; W = W_L + W_F."""
    n, nd = 20, 29
    ang = synth.angles_for(14)
    rng = np.random.default_rng(12)
    x = rng.standard_normal((n, n)); s = rng.standard_normal((14, nd))
    r0, r1, c0, c1 = 3, 11, 5, 18
    M = np.zeros((n, n)); M[r0:r1, c0:c1] = 1
    wl = orc.forward(x, ang, nd, (r0, r1, c0, c1))
    assert np.max(np.abs(wl - orc.forward(M * x, ang, nd))) < 1e-13
    assert np.max(np.abs(wl + orc.forward((1 - M) * x, ang, nd) - orc.forward(x, ang, nd))) < 1e-12
    assert np.max(np.abs(orc.back(s, ang, n, (r0, r1, c0, c1)) - M * orc.back(s, ang, n))) < 1e-13


def test_roi_rects_clip(orc):
    r = orc.roi_rects(64, [[32, 32], [12, 52]], 12, 8)
    assert r[0].tolist() == [20, 44, 20, 44, 12, 52, 12, 52]
    assert r[1].tolist() == [0, 24, 40, 64, 0, 32, 32, 64]
    with pytest.raises(Exception):
        orc.roi_rects(64, [[5, 32]], 12, 8)      # core outside the grid -> error 2


# ---------------------------------------------------------------- SIRT / Alg. 1

def test_P5_sirt_closed_form(orc):
    """P5: x^n = alpha (sum_{k<n} A^k) W^T p, A = I - alpha W^T W (eq. sirtfull2)."""
    n, nd = 8, 13
    ang = synth.angles_for(10)
    W = dense_W(orc, n, ang, nd)
    alpha = 1.0 / (10 * nd)
    p = np.random.default_rng(5).random((10, nd))
    A = np.eye(n * n) - alpha * W.T @ W
    for it in (1, 5, 20):
        S = np.zeros_like(A); Ak = np.eye(n * n)
        for _ in range(it):
            S += Ak; Ak = Ak @ A
        x_cf = alpha * S @ (W.T @ p.ravel())
        x = orc.global_box(p, ang, n, it, lo=-np.inf, hi=np.inf)
        assert relerr(x.ravel(), x_cf) < 1e-10
        if it == 1:
            assert relerr(x.ravel(), alpha * W.T @ p.ravel()) < 1e-13


@pytest.mark.parametrize("n", [8, 9])
def test_P6_filter_bank(orc, n):
    """P6: u_1 = alpha W e_c; u_{k+1} - u_k = alpha W A^k e_c (Alg. 1);
    rows symmetric about d_c; rows of theta and pi - theta equal (symmetric angle set)."""
    nd = 13
    na = 12
    ang = synth.angles_for(na)
    alpha = 1.0 / (na * nd)
    W = dense_W(orc, n, ang, nd)
    A = np.eye(n * n) - alpha * W.T @ W
    ec = np.zeros((n, n))
    if n % 2 == 0:
        m = n // 2; ec[m - 1:m + 1, m - 1:m + 1] = 0.25        # reading A5
    else:
        ec[n // 2, n // 2] = 1.0
    bank = orc.filter_bank(n, ang, nd, 6)
    assert np.max(np.abs(bank[0] - alpha * orc.forward(ec, ang, nd))) < 1e-16
    v = ec.ravel()
    for k in range(1, 6):
        v = A @ v
        assert np.max(np.abs((bank[k] - bank[k - 1]).ravel() - alpha * W @ v)) < 1e-16
    assert np.max(np.abs(bank - bank[:, :, ::-1])) < 1e-15 * np.max(np.abs(bank))
    for a in range(1, na):
        assert np.max(np.abs(bank[:, a] - bank[:, na - a])) < 1e-15 * np.max(np.abs(bank))


def test_P13_filter_approximates_sirt_band(orc):
    """P13 (parity unpinned, tolerance band only): FBP(p, u_n) ~ SIRT_n (eq. sfbp)."""
    cfg = synth.config("C1")
    inp = synth.make_inputs("C1", noise=False)
    p = inp.sino_clean
    bank = orc.filter_bank(64, inp.angles, 91, 50)
    for k in (10, 50):
        fbp = orc.back(orc.convolve(bank[k - 1], p), inp.angles, 64)
        sirt = orc.global_box(p, inp.angles, 64, k, lo=-np.inf, hi=np.inf)
        assert relerr(fbp, sirt) < 0.10


# ---------------------------------------------------------------- convolution / disc

def test_P7_convolution(orc):
    """P7: direct C_h vs numpy convolution; identity filter; linearity."""
    rng = np.random.default_rng(7)
    na, nd = 5, 31
    h = rng.standard_normal((na, nd)); p = rng.standard_normal((na, nd)); q = rng.standard_normal((na, nd))
    out = orc.convolve(h, p)
    dc = (nd - 1) // 2
    for a in range(na):
        ref = np.convolve(h[a], p[a])[dc:dc + nd]
        assert np.max(np.abs(out[a] - ref)) < 1e-12
    ident = np.zeros((na, nd)); ident[:, dc] = 1.0
    assert np.max(np.abs(orc.convolve(ident, p) - p)) == 0.0
    assert np.max(np.abs(orc.convolve(h, 2 * p - 3 * q) - (2 * out - 3 * orc.convolve(h, q)))) < 1e-11


def test_P8_disc(orc):
    """P8: disc correction: p = W D -> c = 1; p = 0 -> c = 0;
    c minimizes the zero-frequency l2 norm over a probe grid; D is the centred disc of diameter N."""
    n, nd = 32, 47
    ang = synth.angles_for(20)
    pc, c, wd, D = orc.disc(np.zeros((20, nd)), ang, n)
    assert c == 0.0
    h = (n - 1) / 2
    jj, ii = np.meshgrid(np.arange(n) - h, h - np.arange(n))
    assert np.array_equal(D, (jj ** 2 + ii ** 2 <= (n / 2) ** 2).astype(float))
    pc, c, _, _ = orc.disc(wd, ang, n)
    assert abs(c - 1.0) < 1e-14 and np.max(np.abs(pc)) < 1e-12
    p = np.random.default_rng(8).random((20, nd)) * 5
    pc, c, wd, _ = orc.disc(p, ang, n)
    P = p.sum(axis=1); Dz = wd.sum(axis=1)
    f = lambda cc: np.sum((P - cc * Dz) ** 2)
    for probe in np.linspace(c - 0.5, c + 0.5, 21):
        assert f(c) <= f(probe) + 1e-9
    assert np.max(np.abs(pc - (p - c * wd))) < 1e-14


# ---------------------------------------------------------------- FGP

def _tv(x):
    return np.abs(np.diff(x, axis=0)).sum() + np.abs(np.diff(x, axis=1)).sum()


def _Lop(P, Q, h, w):
    out = np.zeros((h, w))
    out[:-1, :] += P; out[1:, :] -= P
    out[:, :-1] += Q; out[:, 1:] -= Q
    return out


def test_P11_fgp_duality_gap(orc):
    """P11: the FGP output certifies itself: primal(z) - dual(p,q) >= 0, decreasing
    with iterations, and tiny after many (Beck & Teboulle)."""
    rng = np.random.default_rng(11)
    b = rng.standard_normal((6, 6)); lam = 0.3
    gaps = []
    for it in (10, 100, 1000, 10000):
        x, P, Q = orc.fgp(b, lam, it, return_duals=True)
        assert np.all(np.abs(P) <= 1 + 1e-15) and np.all(np.abs(Q) <= 1 + 1e-15)
        z = b - lam * _Lop(P, Q, 6, 6)
        assert np.max(np.abs(z - x)) < 1e-13
        primal = 0.5 * np.sum((x - b) ** 2) + lam * _tv(x)
        dual = 0.5 * np.sum(b ** 2) - 0.5 * np.sum(z ** 2)
        gaps.append(primal - dual)
    assert all(g >= -1e-12 for g in gaps)
    assert gaps[1] < gaps[0] and gaps[2] < 1e-6 and gaps[3] < 1e-10


def test_P11_fgp_special_cases(orc):
    rng = np.random.default_rng(12)
    b = rng.standard_normal((7, 5))
    assert np.array_equal(orc.fgp(b, 0.0, 10), b)                      # lam = 0 -> identity
    cst = np.full((7, 5), 0.37)
    assert np.max(np.abs(orc.fgp(cst, 0.8, 50) - cst)) < 1e-15          # TV(b) = 0 -> unchanged
    # 1x2 image: prox has the closed form of soft-thresholding the difference
    b2 = np.array([[0.0, 1.0]]); lam = 0.2
    x = orc.fgp(b2, lam, 200)
    assert np.max(np.abs(x - np.array([[0.2, 0.8]]))) < 1e-12


# ---------------------------------------------------------------- local method invariants

def _small_problem(n=16, na=12, seed=9):
    nd = int(math.ceil(math.sqrt(2) * n)) | 1
    ang = synth.angles_for(na)
    shapes = synth.random_shapes(n, 3, 1, np.random.default_rng(seed))
    p = synth.analytic_sinogram(shapes, ang, nd)
    p = p + np.random.default_rng(seed + 1).normal(0, 0.02 * p.max(), p.shape)
    return n, nd, ang, p


def test_P9_split_exactness_box(orc):
    """P9: full-grid ROI, margin 0, x_s^k := exact SIRT iterates -> the local box
    method equals global box-SIRT (eqs. sirtitprior / localmethod)."""
    n, nd, ang, p = _small_problem()
    nk = 15
    _, xs = orc.global_box(p, ang, n, nk, lo=-np.inf, hi=np.inf, iterates=True)
    xg = orc.global_box(p, ang, n, nk, lo=0.0, hi=np.inf)
    cores = orc.local_solve(n, ang, nd, np.zeros((nk, len(ang), nd)), [[n // 2, n // 2]], n // 2, 0,
                            mode="box", lo=0.0, hi=np.inf, xs_exact=xs)
    assert relerr(cores[0], xg) < 1e-12
    assert np.min(xg) >= 0.0 and np.min(cores[0]) >= 0.0


def test_P9_no_clamp_reduces_to_local_fbp(orc):
    """P9b: l = -inf, r = +inf -> y stays 0 and the output is FBP_L(p_c, u_n) + c D (eq. locsirtapp)."""
    n, nd, ang, p = _small_problem(n=20)
    nk = 8
    pc, c, _, D = orc.disc(p, ang, n)
    bank = orc.filter_bank(n, ang, nd, nk)
    b = orc.conv_cache(bank, pc)
    cen = [[9, 11]]; r, m = 4, 3
    cores, ext = orc.local_solve(n, ang, nd, b, cen, r, m, mode="box", lo=-np.inf, hi=np.inf,
                                 disc_c=c, use_disc=True, want_ext=True)
    rect = orc.roi_rects(n, cen, r, m)[0]
    fbp = orc.back(orc.convolve(bank[nk - 1], pc), ang, n, tuple(rect[4:8])) + c * D
    assert relerr(cores[0], fbp[rect[0]:rect[1], rect[2]:rect[3]]) < 1e-12


def test_P10_split_exactness_tv(orc):
    """P10: same split exactness against global FISTA-TV (Alg. 3 corrected, A12);
    lam = 0 without momentum -> x^n = x_s^n."""
    n, nd, ang, p = _small_problem(n=12, na=10)
    nk, lam, nf = 8, 0.02, 30
    _, xs = orc.global_box(p, ang, n, nk, lo=-np.inf, hi=np.inf, iterates=True)
    xg = orc.global_tv(p, ang, n, nk, lam, nf)
    cores = orc.local_solve(n, ang, nd, np.zeros((nk, len(ang), nd)), [[n // 2, n // 2]], n // 2, 0,
                            mode="tv", lam=lam, n_fgp=nf, xs_exact=xs)
    assert relerr(cores[0], xg) < 1e-12
    xg_nomom = orc.global_tv(p, ang, n, nk, lam, nf, momentum=False)
    cores2 = orc.local_solve(n, ang, nd, np.zeros((nk, len(ang), nd)), [[n // 2, n // 2]], n // 2, 0,
                             mode="tv", lam=lam, n_fgp=nf, momentum=False, xs_exact=xs)
    assert relerr(cores2[0], xg_nomom) < 1e-12
    assert relerr(xg, xg_nomom) > 1e-4                      # momentum really changes the iterate
    cores3 = orc.local_solve(n, ang, nd, np.zeros((nk, len(ang), nd)), [[n // 2, n // 2]], n // 2, 0,
                             mode="tv", lam=0.0, n_fgp=nf, momentum=False, xs_exact=xs)
    assert relerr(cores3[0], xs[-1]) < 1e-12


def test_local_y_stays_inside_extended_roi(orc):
    """y is zero outside L' by construction: the ext output is zero outside the valid rect."""
    n, nd, ang, p = _small_problem(n=24)
    bank = orc.filter_bank(n, ang, nd, 5)
    b = orc.conv_cache(bank, p)
    cores, ext = orc.local_solve(n, ang, nd, b, [[5, 19]], 4, 3, mode="box", want_ext=True)
    rect = orc.roi_rects(n, [[5, 19]], 4, 3)[0]
    H, Wd = rect[5] - rect[4], rect[7] - rect[6]
    assert np.all(ext[0][H:, :] == 0) and np.all(ext[0][:, Wd:] == 0)
    assert np.min(cores) >= 0.0


def test_P14_stitch(orc):
    """P14: disjoint tiling -> placement; overlaps -> mean (A19)."""
    n, r = 16, 4
    cen = np.array([[4, 4], [4, 12], [12, 4], [12, 12]])
    cores = np.random.default_rng(14).random((4, 8, 8))
    img = orc.stitch(n, cen, r, cores)
    assert np.array_equal(img[:8, 8:], cores[1]) and np.array_equal(img[8:, :8], cores[2])
    cen2 = np.array([[4, 4], [6, 6]])
    img2 = orc.stitch(n, cen2, r, cores[:2])
    assert img2[3, 3] == 0.5 * (cores[0][3, 3] + cores[1][1, 1])
    assert img2[0, 0] == cores[0][0, 0] and img2[15, 15] == 0.0


# ------------------------------------------------------------------ NEXT-3: truncated data

def test_pad_truncated_pins(orc):
    """Truncated data (constant padding L1148): identity when
    nothing is truncated, zeros stay zeros, the edge value extends each row."""
    rng = np.random.default_rng(31)
    p = rng.random((5, 9))
    assert np.array_equal(orc.pad_truncated(p, 9), p)
    assert np.array_equal(orc.pad_truncated(np.zeros((3, 5)), 11), np.zeros((3, 11)))
    q = orc.pad_truncated(p, 15)
    assert np.array_equal(q[:, 3:12], p)
    assert np.array_equal(q[:, :3], np.repeat(p[:, :1], 3, axis=1))
    assert np.array_equal(q[:, 12:], np.repeat(p[:, -1:], 3, axis=1))
    with pytest.raises(orc.OracleError):
        orc.pad_truncated(p, 10)          # odd difference: no centred padding
    with pytest.raises(orc.OracleError):
        orc.pad_truncated(p, 7)           # target smaller than the data


def test_pad_truncated_keeps_detector_coordinates(orc):
    """Centring pinned against the geometry (V1: t_d = d - (N_d - 1)/2): the
    analytic sinogram measured on n_trunc central bins equals the central bins of
    the full-detector sinogram, and padding puts them back at the same place."""
    shapes = synth.random_shapes(64, 5, 0, synth.seeded_rng(31, 0))
    ang = synth.angles_for(12)
    full = synth.analytic_sinogram(shapes, ang, 91)
    trunc = synth.analytic_sinogram(shapes, ang, 31)
    assert np.allclose(trunc, full[:, 30:61], rtol=0, atol=1e-12)
    assert np.array_equal(orc.pad_truncated(trunc, 91)[:, 30:61], trunc)


# ------------------------------------------------------------------ NEXT-1: metrics, Nelder-Mead

def test_mse_pins(orc):
    """MSE: a == b -> 0; [0,1] vs [1,1] -> 0.5; offset c -> c^2."""
    a = np.random.default_rng(5).random((7, 9))
    assert orc.mse(a, a) == 0.0
    assert orc.mse(np.array([[0.0, 1.0]]), np.array([[1.0, 1.0]])) == 0.5
    assert abs(orc.mse(a + 0.25, a) - 0.0625) < 1e-15


def test_ssim_pins(orc):
    """SSIM (Wang 2004): ssim(a, a) = 1; symmetric for a fixed L;
    constant images c1, c2 -> (2 c1 c2 + C1) / (c1^2 + c2^2 + C1)."""
    rng = np.random.default_rng(6)
    a = rng.random((24, 30)); b = a + 0.1 * rng.standard_normal(a.shape)
    assert abs(orc.ssim(a, a) - 1.0) < 1e-12
    assert abs(orc.ssim(a, b, data_range=1.0) - orc.ssim(b, a, data_range=1.0)) < 1e-12
    c1, c2, L = 0.3, 0.7, 1.0
    C1 = (0.01 * L) ** 2
    got = orc.ssim(np.full((15, 15), c1), np.full((15, 15), c2), data_range=L)
    assert abs(got - (2 * c1 * c2 + C1) / (c1 ** 2 + c2 ** 2 + C1)) < 1e-12
    assert 0.0 < orc.ssim(b, a) < 1.0


def test_ssim_matches_scipy_filtering(orc):
    """Independent route: the same Wang-2004 statistics by scipy.ndimage Gaussian
    correlation (library filtering, 'valid' positions) agree with the oracle's
    explicit window sums."""
    from scipy import ndimage
    rng = np.random.default_rng(7)
    g = np.clip(rng.random((26, 21)), 0, 1)
    x = g + 0.05 * rng.standard_normal(g.shape)
    w = orc.ssim_window()
    def filt(im):
        return ndimage.correlate(im, w, mode="constant")[5:-5, 5:-5]
    mx, mg = filt(x), filt(g)
    vx, vg, cxg = filt(x * x) - mx ** 2, filt(g * g) - mg ** 2, filt(x * g) - mx * mg
    L = g.max() - g.min()
    C1, C2 = (0.01 * L) ** 2, (0.03 * L) ** 2
    ref = np.mean((2 * mx * mg + C1) * (2 * cxg + C2) / ((mx ** 2 + mg ** 2 + C1) * (vx + vg + C2)))
    assert abs(orc.ssim(x, g) - ref) < 1e-12


def test_nelder_mead_pins(orc):
    """Nelder-Mead in one dimension: finds the minimum of
    (t - 2)^2 within 50 evaluations, honours the budget exactly, never leaves the
    bounds, and a monotone objective ends at the boundary."""
    t, v, n = orc.nelder_mead_1d(lambda t: (t - 2.0) ** 2, -3.0, 4.0, 50)
    assert abs(t - 2.0) < 1e-2 and n <= 50
    calls = []
    t, v, n = orc.nelder_mead_1d(lambda t: calls.append(t) or (t - 2.0) ** 2, -3.0, 4.0, 3)
    assert n == 3 and len(calls) == 3
    seen = []
    t, v, n = orc.nelder_mead_1d(lambda t: seen.append(t) or t, -3.0, 4.0, 40)
    assert all(-3.0 <= s <= 4.0 for s in seen) and t == -3.0


# ------------------------------------------------------------------ NEXT-2: Haar l1 prior

def test_haar_pins(orc):
    """Orthonormal 2D Haar: inverse o forward = identity, Parseval,
    a constant image has the single coefficient c 2^levels, one level on a 2x2
    block is the closed-form orthonormal map, sizes must be divisible."""
    rng = np.random.default_rng(41)
    x = rng.standard_normal((32, 48))
    for L in (1, 3, 4):
        c = orc.haar(x, L)
        assert np.allclose(orc.haar(c, L, inverse=True), x, rtol=0, atol=1e-12)
        assert abs(np.linalg.norm(c) - np.linalg.norm(x)) < 1e-12
    c = orc.haar(np.full((16, 16), 0.7), 4)
    assert abs(c[0, 0] - 0.7 * 16) < 1e-12 and np.count_nonzero(np.abs(c) > 1e-12) == 1
    a, b, cc, d = 1.0, 2.0, 3.0, 5.0
    got = orc.haar(np.array([[a, b], [cc, d]]), 1)
    assert np.allclose(got, 0.5 * np.array([[a + b + cc + d, a - b + cc - d], [a + b - cc - d, a - b - cc + d]]),
                       rtol=0, atol=1e-15)
    with pytest.raises(orc.OracleError):
        orc.haar(np.zeros((12, 16)), 3)


def test_haar_prox_pins(orc):
    """P_lambda (symmetric reading A15): lambda = 0 is the
    identity; the prox equals the closed-form minimiser of 1/2||x - v||^2 +
    lambda ||Bx||_1 (componentwise in the orthonormal basis): checked by
    optimality - no single-coefficient perturbation lowers the objective."""
    rng = np.random.default_rng(42)
    v = rng.standard_normal((16, 16))
    assert np.allclose(orc.haar_prox(v, 0.0, 4), v, rtol=0, atol=1e-12)
    lam = 0.3
    x = orc.haar_prox(v, lam, 2)
    def obj(z):
        return 0.5 * np.sum((z - v) ** 2) + lam * np.sum(np.abs(orc.haar(z, 2)))
    f0 = obj(x)
    cx = orc.haar(x, 2)
    for (i, j) in [(0, 0), (1, 3), (5, 7), (15, 15)]:
        for eps in (1e-4, -1e-4):
            c2 = cx.copy(); c2[i, j] += eps
            assert obj(orc.haar(c2, 2, inverse=True)) >= f0 - 1e-12
    assert np.all(np.abs(orc.haar(orc.haar_prox(v, 10.0, 2), 2)) == 0.0)   # lambda above every |coefficient|


def test_local_haar_lambda0_equals_unregularized(orc):
    """Haar prior with lambda = 0 is the identity prox: the local Haar-FISTA path
    equals the local TV path with lambda = 0 (both plain FISTA on S)."""
    n, nd, ang, p = _small_problem(n=24)
    bank = orc.filter_bank(n, ang, nd, 6)
    b = orc.conv_cache(bank, p)
    cen = [[12, 12]]
    a = orc.local_solve(n, ang, nd, b, cen, 4, 4, mode="haar", lam=0.0, levels=3)
    t = orc.local_solve(n, ang, nd, b, cen, 4, 4, mode="tv", lam=0.0, n_fgp=10)
    assert relerr(a, t) < 1e-13


# ------------------------------------------------------------------ NEXT-4(iii): Chambolle-Pock TV

def _cp_problem():
    n, nd = 8, 13
    ang = synth.angles_for(32)          # W has full column rank (condition number ~50)
    shapes = synth.random_shapes(n, 2, 0, synth.seeded_rng(11, 0))
    return n, nd, ang, synth.analytic_sinogram(shapes, ang, nd)


def test_cp_mu0_is_least_squares(orc):
    """mu = 0: preconditioned CP minimises 1/2||Wx - p||^2; W has full column rank
    here, so it converges to the unique least-squares solution (numpy lstsq of
    the dense W assembled column by column from the oracle's W)."""
    n, nd, ang, p = _cp_problem()
    Wd = np.stack([orc.forward(np.eye(n * n)[k].reshape(n, n), ang, nd).ravel() for k in range(n * n)], axis=1)
    assert np.linalg.matrix_rank(Wd) == n * n
    ls = np.linalg.lstsq(Wd, p.ravel(), rcond=None)[0].reshape(n, n)
    x = orc.global_cp(p, ang, n, 10000, 0.0)
    assert relerr(x, ls) < 1e-10


def test_cp_reaches_the_fista_tv_minimiser(orc):
    """Same objective as global FISTA-TV (reading A14: mu = lam / alpha): both
    converge to the unique minimiser of the strictly convex problem; CP (exact
    proximal steps) ends no higher than FISTA with its inexact 300-step FGP prox."""
    n, nd, ang, p = _cp_problem()
    alpha = 1.0 / (len(ang) * nd)
    lam = 0.002
    mu = lam / alpha
    def F(x):
        r = orc.forward(x, ang, nd) - p
        return 0.5 * np.sum(r * r) + mu * (np.abs(np.diff(x, axis=0)).sum() + np.abs(np.diff(x, axis=1)).sum())
    xf = orc.global_tv(p, ang, n, 3000, lam, 300)
    xc = orc.global_cp(p, ang, n, 30000, mu)
    assert F(xc) <= F(xf) * (1 + 1e-12)
    assert abs(F(xc) - F(xf)) <= 1e-5 * F(xf)
    assert relerr(xc, xf) < 1e-4


# ------------------------------------------------------------------ NEXT-4(ii): exterior subtraction

def test_exterior_full_grid_is_global_box_sirt(orc):
    """A ROI covering the grid has no exterior (M_F = 0): whatever the
    global reconstruction, the exterior-subtraction solve is global box-SIRT."""
    n, nd, ang, p = _small_problem(n=16)
    xg = np.random.default_rng(3).random((n, n))
    cores = orc.exterior_solve(p, ang, n, xg, [[8, 8]], 8, 0, 12)
    ref = orc.global_box(p, ang, n, 12)
    assert relerr(cores[0], ref) < 1e-12


def test_exterior_with_exact_exterior_is_local_sirt_of_the_roi_data(orc):
    """With consistent data p = W x_true and xg = x_true, p - W M_F xg = W M_L' x_true:
    the ROI solve is box-SIRT on L' for data generated by the ROI part alone
    (checked against global box-SIRT of the masked object restricted to L')."""
    n, nd = 16, 23
    ang = synth.angles_for(14)
    xt = np.random.default_rng(4).random((n, n))
    p = orc.forward(xt, ang, nd)
    cen, r, m = [[8, 7]], 3, 2
    rect = orc.roi_rects(n, cen, r, m)[0]
    cores = orc.exterior_solve(p, ang, n, xt, cen, r, m, 10, lo=-np.inf, hi=np.inf)
    # the same iteration written with the global operators and the mask
    M = np.zeros((n, n)); M[rect[4]:rect[5], rect[6]:rect[7]] = 1.0
    pl = orc.forward(M * xt, ang, nd)
    x = np.zeros((n, n)); alpha = orc.alpha_for(len(ang), nd)
    for _ in range(10):
        x = x + alpha * M * orc.back(pl - orc.forward(M * x, ang, nd), ang, n)
    assert relerr(cores[0], x[rect[0]:rect[1], rect[2]:rect[3]]) < 1e-12


# ------------------------------------------------------------------ eq. localmethod off the grid origin, FISTA beta

def _fista_table():
    """tests/golden/fista_tk.txt: k, t_k, beta_k (Beck & Teboulle 2009, written by make_fista_tk.py)."""
    rows = [l.split() for l in open(os.path.join(GOLDEN, "fista_tk.txt")) if l.strip() and not l.startswith("#")]
    k = np.array([int(r[0]) for r in rows])
    t = np.array([float(r[1]) for r in rows])
    b = np.array([float(r[2]) for r in rows])
    return k, t, b


def test_fista_table_is_beck_teboulle():
    """The golden FISTA sequence has the properties that define it (Beck & Teboulle
    2009, cited at P:L660; Alg. 3 P:L679-680 corrected per A12): t_1 = 1, t_2 = the
    golden ratio, t_{k+1}^2 - t_{k+1} = t_k^2 (the quadratic whose root the update
    takes), t_k >= (k+1)/2 (their Lemma 4.3), beta_1 = 0, 0 < beta_k < 1 increasing."""
    k, t, b = _fista_table()
    assert k[0] == 1 and t[0] == 1.0 and b[0] == 0.0
    assert abs(t[1] - (1.0 + math.sqrt(5.0)) / 2.0) < 1e-15
    assert np.all(np.abs(t[1:] ** 2 - t[1:] - t[:-1] ** 2) <= 1e-13 * t[1:] ** 2)
    assert np.all(t >= (k + 1) / 2.0 - 1e-15)
    assert np.all(np.diff(b) > 0) and np.all(b[1:] > 0) and np.all(b < 1)
    assert np.all(np.abs(b[:-1] * t[1:] - (t[:-1] - 1.0)) < 1e-13 * t[1:])


@pytest.mark.parametrize("mode", ["box", "tv"])
def test_local_recursion_off_origin_equals_masked_global_operators(orc, mode):
    """eq. localmethod / Alg. 2 / Alg. 3 on a
    CLIPPED, OFF-CENTRE extended ROI (rows start at the grid edge, columns at 11,
    non-square) with noisy data and the disc term, written with the already-pinned
    global operators and the mask M_{L'} (W_{L'} = W M_{L'}, W_{L'}^T = M_{L'} W^T,
    P:L250-251, pin P12):
        x_s^k = M W^T b_k + c M D                              (A7)
        S     = x_s^k + y - alpha M W^T W M y
        box:  x = clamp(S), y = x - x_s^k
        TV:   x = FGP(S on L'), r = x + beta_k (x - x_prev), y = r - x_s^k
              with beta_k from the golden Beck-Teboulle table (A12)
    The oracle's windowless local solve must agree to 1e-12; a swapped row/column
    offset of the y projection, or a wrong momentum sequence, fails here."""
    n, nd, ang, p = _small_problem(n=24, na=14, seed=21)
    nk, lam, nf = 9, 0.03, 25
    pc, c, _, D = orc.disc(p, ang, n)
    bank = orc.filter_bank(n, ang, nd, nk)
    b = orc.conv_cache(bank, pc)
    cen, r, m = [[5, 18]], 4, 3
    rect = orc.roi_rects(n, cen, r, m)[0]
    er0, er1, ec0, ec1 = (int(v) for v in rect[4:8])
    assert (er0, er1, ec0, ec1) == (0, 12, 11, 24)        # clipped on two sides, off the origin, 12 x 13
    R = (er0, er1, ec0, ec1)
    M = np.zeros((n, n)); M[er0:er1, ec0:ec1] = 1.0
    alpha = orc.alpha_for(len(ang), nd)
    _, _, beta = _fista_table()
    y = np.zeros((n, n)); xprev = np.zeros((n, n)); x = np.zeros((n, n))
    for k in range(nk):
        xs = orc.back(b[k], ang, n, R) + c * M * D
        S = xs + y - alpha * orc.back(orc.forward(y, ang, nd, R), ang, n, R)
        if mode == "box":
            x = M * np.clip(S, 0.0, np.inf)
            y = x - xs
        else:
            x = np.zeros((n, n))
            x[er0:er1, ec0:ec1] = orc.fgp(S[er0:er1, ec0:ec1], lam, nf)
            y = x + beta[k] * (x - xprev) - xs
            xprev = x
    cores = orc.local_solve(n, ang, nd, b, cen, r, m, mode=mode, lo=0.0, hi=np.inf, lam=lam, n_fgp=nf,
                            disc_c=c, use_disc=True)
    ref = x[rect[0]:rect[1], rect[2]:rect[3]]
    assert relerr(cores[0], ref) < 1e-12
    if mode == "box":
        assert np.min(S) < 0.0                            # the clamp was active
    assert np.max(np.abs(y * (1 - M))) == 0.0             # y stays inside L'


def test_fista_momentum_follows_the_golden_sequence(orc):
    """Alg. 3 with lambda = 0 (FGP = identity), a full-grid ROI and the exact SIRT
    iterates as x_s is FISTA on 1/2||p - Wx||^2 with step alpha (split
    exactness P9/P10): x^k = r^{k-1} + alpha W^T (p - W r^{k-1}),
    r^k = x^k + beta_k (x^k - x^{k-1}), beta_k from tests/golden/fista_tk.txt.
    Both the local solve and the global FISTA-TV of the oracle must follow it to
    1e-12 (a beta of (t'-1)/(t'+1), or t_{k} in place of t_{k-1}, fails)."""
    n, nd, ang, p = _small_problem(n=12, na=10, seed=5)
    nk = 14
    alpha = orc.alpha_for(len(ang), nd)
    _, _, beta = _fista_table()
    x = np.zeros((n, n)); r_ = np.zeros((n, n))
    for k in range(nk):
        xn = r_ + alpha * orc.back(p - orc.forward(r_, ang, nd), ang, n)
        r_ = xn + beta[k] * (xn - x)
        x = xn
    _, xs = orc.global_box(p, ang, n, nk, lo=-np.inf, hi=np.inf, iterates=True)
    cores = orc.local_solve(n, ang, nd, np.zeros((nk, len(ang), nd)), [[n // 2, n // 2]], n // 2, 0,
                            mode="tv", lam=0.0, n_fgp=1, xs_exact=xs)
    assert relerr(cores[0], x) < 1e-12
    assert relerr(orc.global_tv(p, ang, n, nk, 0.0, 1), x) < 1e-12
    assert relerr(x, xs[-1]) > 1e-3                       # momentum really changes the iterate


def test_fgp_iterates_follow_beck_teboulle(orc):
    """The FGP (Beck & Teboulle 2009, named at P:L661-663; reading A13) step by
    step on a ragged 5 x 7 image: dual step 1/(8 lambda), projection onto [-1, 1],
    momentum beta_k from the golden table, output b - lambda L(p, q); oracle
    iterates for n_FGP = 1, 2, 3, 7, 20 agree to 1e-12 (the inner momentum is
    otherwise pinned only by convergence, P11)."""
    rng = np.random.default_rng(11)
    bimg = rng.random((5, 7))
    lam = 0.07
    _, _, beta = _fista_table()
    h, w = bimg.shape

    def Lop(P, Q):
        out = np.zeros((h, w))
        out[:-1, :] += P; out[1:, :] -= P
        out[:, :-1] += Q; out[:, 1:] -= Q
        return out

    for nit in (1, 2, 3, 7, 20):
        P = np.zeros((h - 1, w)); Q = np.zeros((h, w - 1)); Rr = P.copy(); Ss = Q.copy()
        for it in range(nit):
            z = bimg - lam * Lop(Rr, Ss)
            Pn = np.clip(Rr + (z[:-1, :] - z[1:, :]) / (8 * lam), -1, 1)
            Qn = np.clip(Ss + (z[:, :-1] - z[:, 1:]) / (8 * lam), -1, 1)
            Rr = Pn + beta[it] * (Pn - P); Ss = Qn + beta[it] * (Qn - Q)
            P, Q = Pn, Qn
        x = bimg - lam * Lop(P, Q)
        assert relerr(orc.fgp(bimg, lam, nit), x) < 1e-12, nit
