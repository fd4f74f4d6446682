"""fp64 CPU oracle for the local approximation of regularized iterative
tomography (Pelt & Batenburg, arXiv 1604.02292).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
package.  The product package ``paper_1604_02292_b200`` never imports it and
the two share no code.

The arithmetic lives in ``loctomo_oracle.c`` (plain C, fp64, OpenMP over
independent outputs only); this module is ctypes marshalling plus
``build()``.  Every C entry point cites the PAPER.md passage it follows.

Parity status: every function here is pinned by tests/test_oracle_pins.py
except the approximation-quality comparisons (FBP(p,u_n) vs SIRT_n, local vs
global), which are "parity unpinned" by nature (tolerance bands only, P13 in
DESIGN.md).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "loctomo_oracle.c")
_LIB_PATH = os.path.join(_HERE, "_loctomo_oracle.so")
_lib = None

OK, ERR_RUNTIME, ERR_INVALID = 0, 1, 2


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc, -O2 -msse4.1, OpenMP, no -ffast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        # -msse4.1: floor/ceil as single instructions (no libm calls); the
        # arithmetic is unchanged (no -ffast-math, results bitwise identical)
        cmd = ["gcc", "-O2", "-msse4.1", "-std=gnu11", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
               _SRC, "-o", _LIB_PATH + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


def _L():
    global _lib
    if _lib is None:
        alt = os.environ.get("LT_ORACLE_SO")     # mutation testing only (tools/oracle_mutants.py)
        if alt:
            _lib = ctypes.CDLL(alt)
        else:
            build()
            _lib = ctypes.CDLL(_LIB_PATH)
    return _lib


def _d(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _chk(rc: int, what: str):
    if rc != OK:
        raise OracleError(f"{what} failed with code {rc}")


def set_threads(n: int) -> None:
    _L().or_set_threads(ctypes.c_int(int(n)))


def get_threads() -> int:
    return int(_L().or_get_threads())


def alpha_for(n_angles: int, n_det: int) -> float:
    """alpha = (N_theta N_d)^-1."""
    return 1.0 / (n_angles * n_det)


def forward(img: np.ndarray, angles, n_det: int, rect: Optional[Tuple[int, int, int, int]] = None) -> np.ndarray:
    """W M_R x (rect = (r0, r1, c0, c1), default the full grid).  PAPER.md L244, L250."""
    img = _f64(img)
    n = img.shape[0]
    ang = _f64(angles)
    r0, r1, c0, c1 = (int(v) for v in rect) if rect is not None else (0, n, 0, n)
    out = np.zeros((len(ang), n_det))
    _chk(_L().or_forward(n, len(ang), n_det, _d(ang), _d(img), r0, r1, c0, c1, _d(out)), "or_forward")
    return out


def back(sino: np.ndarray, angles, n: int, rect: Optional[Tuple[int, int, int, int]] = None) -> np.ndarray:
    """M_R W^T s on the N x N grid.  PAPER.md L244, L251."""
    sino = _f64(sino)
    ang = _f64(angles)
    r0, r1, c0, c1 = (int(v) for v in rect) if rect is not None else (0, n, 0, n)
    out = np.zeros((n, n))
    _chk(_L().or_back(n, len(ang), sino.shape[1], _d(ang), _d(sino), r0, r1, c0, c1, _d(out)), "or_back")
    return out


def filter_bank(n: int, angles, n_det: int, n_k: int, alpha: Optional[float] = None) -> np.ndarray:
    """Alg. 1 with every u_k kept: [n_k, N_theta, N_d].  PAPER.md L489-503, L621-624."""
    ang = _f64(angles)
    a = alpha_for(len(ang), n_det) if alpha is None else alpha
    out = np.zeros((n_k, len(ang), n_det))
    _chk(_L().or_filter_bank(n, len(ang), n_det, _d(ang), n_k, ctypes.c_double(a), _d(out)), "or_filter_bank")
    return out


def convolve(h: np.ndarray, p: np.ndarray) -> np.ndarray:
    """C_h p per detector row, centre aligned."""
    h = _f64(h); p = _f64(p)
    out = np.zeros_like(p)
    _chk(_L().or_convolve(p.shape[0], p.shape[1], _d(h), _d(p), _d(out)), "or_convolve")
    return out


def conv_cache(bank: np.ndarray, p: np.ndarray) -> np.ndarray:
    """b_k = C_{u_k} p for every k."""
    return np.stack([convolve(bank[k], p) for k in range(bank.shape[0])])


def disc(p: np.ndarray, angles, n: int):
    """Disc pre-correction.  Returns (p_c, c, W D, D)."""
    p = _f64(p); ang = _f64(angles)
    pc = np.zeros_like(p); wd = np.zeros_like(p); dimg = np.zeros((n, n))
    c = ctypes.c_double(0.0)
    _chk(_L().or_disc(n, len(ang), p.shape[1], _d(ang), _d(p), _d(pc), ctypes.byref(c), _d(wd), _d(dimg)), "or_disc")
    return pc, c.value, wd, dimg


def fgp(b: np.ndarray, lam: float, n_iter: int, return_duals: bool = False):
    """FGP TV prox (Beck & Teboulle), anisotropic, Neumann."""
    b = _f64(b)
    h, w = b.shape
    x = np.zeros_like(b)
    P = np.zeros((max(h - 1, 0), w)); Q = np.zeros((h, max(w - 1, 0)))
    _chk(_L().or_fgp(h, w, _d(b), ctypes.c_double(lam), n_iter, _d(x),
                     _d(P) if P.size else None, _d(Q) if Q.size else None), "or_fgp")
    return (x, P, Q) if return_duals else x


def haar(x: np.ndarray, levels: int, inverse: bool = False) -> np.ndarray:
    """Orthonormal 2D Haar, in-place layout (NEXT-2; "wavelet decomposition
    operator B", Haar basis L764)."""
    y = np.ascontiguousarray(_f64(x)).copy()
    _chk(_L().or_haar(y.shape[0], y.shape[1], levels, int(inverse), _d(y)), "or_haar")
    return y


def haar_prox(v: np.ndarray, lam: float, levels: int) -> np.ndarray:
    """B^{-1} P_lambda(B v) with the symmetric soft threshold (eq. sirtista, A15)."""
    v = np.ascontiguousarray(_f64(v))
    x = np.zeros_like(v)
    _chk(_L().or_haar_prox(v.shape[0], v.shape[1], levels, _d(v), ctypes.c_double(lam), _d(x)), "or_haar_prox")
    return x


def roi_rects(n: int, centres, radius: int, margin: int) -> np.ndarray:
    """[R, 8] = core (r0, r1, c0, c1), extended (r0, r1, c0, c1)."""
    c = _i32(centres).reshape(-1, 2)
    out = np.zeros((c.shape[0], 8), dtype=np.int32)
    _chk(_L().or_roi_rects(n, c.shape[0], _i(c), radius, margin, _i(out)), "or_roi_rects")
    return out


def local_solve(n: int, angles, n_det: int, bconv: np.ndarray, centres, radius: int, margin: int,
                mode: str = "box", lo: float = 0.0, hi: float = np.inf, lam: float = 0.0,
                n_fgp: int = 100, momentum: bool = True, disc_c: float = 0.0, use_disc: bool = False,
                alpha: Optional[float] = None, xs_exact: Optional[np.ndarray] = None,
                want_ext: bool = False, levels: int = 4):
    """Alg. 2 (box) / Alg. 3 (TV; "haar": the Haar l1 prior, NEXT-2, `levels`
    levels) for every ROI.  Returns cores [R, 2r, 2r] (and ext [R, 2h, 2h]
    when want_ext).  PAPER.md L613-620, L637-688."""
    ang = _f64(angles)
    bconv = _f64(bconv)
    nk = bconv.shape[0]
    a = alpha_for(len(ang), n_det) if alpha is None else alpha
    c = _i32(centres).reshape(-1, 2)
    R = c.shape[0]
    side, eside = 2 * radius, 2 * (radius + margin)
    cores = np.zeros((R, side, side))
    ext = np.zeros((R, eside, eside)) if want_ext else None
    xe = _f64(xs_exact) if xs_exact is not None else None
    rc = _L().or_local_solve(n, len(ang), n_det, _d(ang), nk, ctypes.c_double(a), _d(bconv),
                             ctypes.c_double(disc_c), int(use_disc), R, _i(c), radius, margin,
                             {"box": 0, "tv": 1, "haar": 2}[mode], ctypes.c_double(lo), ctypes.c_double(hi),
                             ctypes.c_double(lam), levels if mode == "haar" else n_fgp, int(momentum),
                             _d(xe) if xe is not None else None, _d(cores),
                             _d(ext) if ext is not None else None)
    _chk(rc, "or_local_solve")
    return (cores, ext) if want_ext else cores


def global_box(p: np.ndarray, angles, n: int, n_iter: int, lo: float = 0.0, hi: float = np.inf,
               alpha: Optional[float] = None, iterates: bool = False):
    """Box-constrained SIRT on the full grid."""
    p = _f64(p); ang = _f64(angles)
    a = alpha_for(len(ang), p.shape[1]) if alpha is None else alpha
    x = np.zeros((n, n))
    it = np.zeros((n_iter, n, n)) if iterates else None
    _chk(_L().or_global_box(n, len(ang), p.shape[1], _d(ang), _d(p), n_iter, ctypes.c_double(a),
                            ctypes.c_double(lo), ctypes.c_double(hi), _d(x),
                            _d(it) if it is not None else None), "or_global_box")
    return (x, it) if iterates else x


def global_tv(p: np.ndarray, angles, n: int, n_iter: int, lam: float, n_fgp: int = 100,
              momentum: bool = True, alpha: Optional[float] = None) -> np.ndarray:
    """FISTA-TV with FGP prox on the full grid (reading A12/A14)."""
    p = _f64(p); ang = _f64(angles)
    a = alpha_for(len(ang), p.shape[1]) if alpha is None else alpha
    x = np.zeros((n, n))
    _chk(_L().or_global_tv(n, len(ang), p.shape[1], _d(ang), _d(p), n_iter, ctypes.c_double(a),
                           ctypes.c_double(lam), n_fgp, int(momentum), _d(x)), "or_global_tv")
    return x


def exterior_solve(p: np.ndarray, angles, n: int, xg: np.ndarray, centres, radius: int, margin: int,
                   n_iter: int, lo: float = 0.0, hi: float = np.inf, alpha: Optional[float] = None) -> np.ndarray:
    """Exterior subtraction (prior art; NEXT-4(ii)): box-SIRT on
    each extended ROI with the data p - W M_F xg.  Returns cores [R, 2r, 2r]."""
    p = _f64(p); ang = _f64(angles); xg = np.ascontiguousarray(_f64(xg))
    a = alpha_for(len(ang), p.shape[1]) if alpha is None else alpha
    c = _i32(centres).reshape(-1, 2)
    cores = np.zeros((c.shape[0], 2 * radius, 2 * radius))
    _chk(_L().or_exterior_solve(n, len(ang), p.shape[1], _d(ang), _d(p), _d(xg), c.shape[0], _i(c), radius, margin,
                                n_iter, ctypes.c_double(a), ctypes.c_double(lo), ctypes.c_double(hi), _d(cores)),
         "or_exterior_solve")
    return cores


def fbp_filtered(p: np.ndarray, angles, n: int, n_k: int, use_disc: bool = True,
                 bank: Optional[np.ndarray] = None) -> np.ndarray:
    """Global FBP with the SIRT-approximating filter u_{n_k} (eq. sfbp P:L481-485,
    Alg. 1) plus the disc correction: x = W^T C_{u_n} p_c + c D."""
    p = _f64(p)
    nd = p.shape[1]
    if use_disc:
        pc, c, _, D = disc(p, angles, n)
    else:
        pc, c, D = p, 0.0, np.zeros((n, n))
    if bank is None:
        bank = filter_bank(n, angles, nd, n_k)
    return back(convolve(bank[n_k - 1], pc), angles, n) + c * D


def global_cp(p: np.ndarray, angles, n: int, n_iter: int, mu: float) -> np.ndarray:
    """Chambolle-Pock TV with diagonal (row / column sum) preconditioning on the
    full grid, minimising 1/2||Wx - p||^2 + mu ||grad x||_1 (NEXT-4(iii))."""
    p = _f64(p); ang = _f64(angles)
    x = np.zeros((n, n))
    _chk(_L().or_global_cp(n, len(ang), p.shape[1], _d(ang), _d(p), n_iter, ctypes.c_double(mu), _d(x)),
         "or_global_cp")
    return x


def stitch(n: int, centres, radius: int, cores: np.ndarray) -> np.ndarray:
    """Mean over covering cores, ascending ROI order (A19)."""
    c = _i32(centres).reshape(-1, 2)
    cores = _f64(cores)
    img = np.zeros((n, n))
    _chk(_L().or_stitch(n, c.shape[0], _i(c), radius, _d(cores), _d(img)), "or_stitch")
    return img


def pad_truncated(p_t: np.ndarray, n_det: int) -> np.ndarray:
    """Truncated projection data:
    each angle row of the n_trunc measured central bins is extended on both
    sides with its edge value ("constant padding", L1148) to n_det bins, centred
    so that bin j of the truncated row keeps its detector coordinate."""
    p_t = _f64(p_t)
    na, nt = p_t.shape
    if nt < 1 or n_det < nt or (n_det - nt) % 2:
        raise OracleError("pad_truncated: need 1 <= n_trunc <= n_det, n_det - n_trunc even")
    lo = (n_det - nt) // 2
    out = np.empty((na, n_det))
    for a in range(na):
        out[a, :lo] = p_t[a, 0]
        out[a, lo:lo + nt] = p_t[a]
        out[a, lo + nt:] = p_t[a, nt - 1]
    return out


def pipeline(p: np.ndarray, angles, n: int, centres, radius: int, margin: int, n_iter: int,
             mode: str = "box", lo: float = 0.0, hi: float = np.inf, lam: float = 0.0,
             n_fgp: int = 100, use_disc: bool = True, bank: Optional[np.ndarray] = None,
             want_ext: bool = False, levels: int = 4):
    """The whole local path for a set of ROIs: disc (a2) -> bank (a3) ->
    conv cache (a4) -> local iterations (a5-a8) -> cores (a9 crop)."""
    p = _f64(p)
    n_det = p.shape[1]
    if use_disc:
        pc, c, _, _ = disc(p, angles, n)
    else:
        pc, c = p, 0.0
    if bank is None:
        bank = filter_bank(n, angles, n_det, n_iter)
    b = conv_cache(bank[:n_iter], pc)
    return local_solve(n, angles, n_det, b, centres, radius, margin, mode=mode, lo=lo, hi=hi,
                       lam=lam, n_fgp=n_fgp, disc_c=c, use_disc=use_disc, want_ext=want_ext, levels=levels)


# --------------------------------------------------------------------------- NEXT-1: metrics, Nelder-Mead

def mse(x: np.ndarray, ref: np.ndarray) -> float:
    """Mean squared error inside the region."""
    x = _f64(x); ref = _f64(ref)
    if x.shape != ref.shape:
        raise OracleError("size mismatch")
    return float(np.mean((x - ref) ** 2))


def ssim_window() -> np.ndarray:
    """11 x 11 Gaussian window, sigma 1.5, normalised (Wang et al. 2004)."""
    a = np.arange(11) - 5.0
    w = np.exp(-(a[:, None] ** 2 + a[None, :] ** 2) / (2.0 * 1.5 ** 2))
    return w / w.sum()


def ssim(x: np.ndarray, ref: np.ndarray, data_range: Optional[float] = None) -> float:
    """Mean SSIM (Wang et al. 2004): at every position where the
    11 x 11 window lies inside the image, with population moments under the
    window weights, C1 = (0.01 L)^2, C2 = (0.03 L)^2, L = max ref - min ref."""
    x = _f64(x); g = _f64(ref)
    if x.shape != g.shape:
        raise OracleError("size mismatch")
    L = float(data_range) if data_range else float(g.max() - g.min())
    C1, C2 = (0.01 * L) ** 2, (0.03 * L) ** 2
    w = ssim_window()
    h, wd = x.shape
    vals = []
    for i in range(h - 10):
        for j in range(wd - 10):
            xa = x[i:i + 11, j:j + 11]; ga = g[i:i + 11, j:j + 11]
            mx, mg = np.sum(w * xa), np.sum(w * ga)
            vx = np.sum(w * xa * xa) - mx * mx
            vg = np.sum(w * ga * ga) - mg * mg
            cxg = np.sum(w * xa * ga) - mx * mg
            vals.append((2 * mx * mg + C1) * (2 * cxg + C2) / ((mx * mx + mg * mg + C1) * (vx + vg + C2)))
    return float(np.mean(vals)) if vals else 0.0


def nelder_mead_1d(f, t_lo: float, t_hi: float, budget: int):
    """Nelder & Mead (1965) in one dimension: initial simplex
    {mid, mid + 0.5}, reflection 1, expansion 2, contraction 1/2, shrink 1/2,
    trial points clamped into [t_lo, t_hi], at most `budget` evaluations.
    Returns (t_best, f_best, evaluations)."""
    if not t_lo < t_hi or budget < 3:
        raise OracleError("need t_lo < t_hi and budget >= 3")
    state = {"n": 0, "bx": None, "bf": math.inf}

    def clamp(t):
        return min(max(t, t_lo), t_hi)

    def F(t):
        t = clamp(t)
        v = f(t)
        state["n"] += 1
        if state["n"] == 1 or v < state["bf"]:
            state["bf"], state["bx"] = v, t
        return v

    mid = 0.5 * (t_lo + t_hi)
    x0, x1 = mid, clamp(mid + 0.5)
    if x1 == x0:
        x1 = clamp(mid - 0.5)
    f0, f1 = F(x0), F(x1)
    while state["n"] < budget:
        if f1 < f0:
            x0, x1, f0, f1 = x1, x0, f1, f0
        if abs(x1 - x0) < 1e-9:
            break
        xr = clamp(x0 + (x0 - x1))
        fr = F(xr)
        if fr < f0:
            if state["n"] < budget:
                xe = clamp(x0 + 2.0 * (xr - x0))
                fe = F(xe)
                x1, f1 = (xe, fe) if fe < fr else (xr, fr)
            else:
                x1, f1 = xr, fr
            continue
        if state["n"] >= budget:
            break
        if fr < f1:
            xc = clamp(x0 + 0.5 * (xr - x0))
            fc = F(xc)
            if fc <= fr:
                x1, f1 = xc, fc
                continue
        else:
            xc = clamp(x0 + 0.5 * (x1 - x0))
            fc = F(xc)
            if fc < f1:
                x1, f1 = xc, fc
                continue
        if state["n"] >= budget:
            break
        x1 = x0 + 0.5 * (x1 - x0)
        f1 = F(x1)
    return state["bx"], state["bf"], state["n"]
