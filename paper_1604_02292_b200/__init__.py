"""B200-native local approximation of regularized iterative tomography
(Pelt & Batenburg, arXiv 1604.02292).

Thin ctypes binding over the C-ABI library ``_loctomo.so`` (declared in
``include/loctomo.h``): argument marshalling only -- every step of the path
runs in the library's sm_100a kernels.  PyTorch provides device memory and
streams.  There is no CPU fallback: importing this package without the built
extension raises, and every call requires CUDA tensors.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional, Sequence

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_loctomo.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the CUDA extension is required; there is no fallback)")

_lib = ctypes.CDLL(LIB_PATH)

LT_OK, LT_ERR_RUNTIME, LT_ERR_INVALID = 0, 1, 2
LT_DISC_ON = 1
LT_XS_EXACT = 2

_P = ctypes.c_void_p
_I = ctypes.c_int32
_F = ctypes.c_float
_i64 = ctypes.c_int64

_SIGS = {
    "lt_roi_setup": ([_I, _I, _I, _P, _I, _P, _P, _I, _I, _I, _I, _I, _I, _P], _I),
    "lt_plan_workspace_bytes": ([_P], _i64),
    "lt_plan_bind_workspace": ([_P, _P, _i64, _P], _I),
    "lt_plan_local_count": ([_P], _I),
    "lt_plan_local_rois": ([_P, _P], _I),
    "lt_plan_tables": ([_P, _P, _P, _P], _I),
    "lt_filter_bank": ([_P, _P], _I),
    "lt_set_bank": ([_P, _P, _P], _I),
    "lt_bank_split_begin": ([_P, _I, _I, _P], _I),
    "lt_bank_split_step": ([_P, _I, _P, _P], _I),
    "lt_bank_split_apply": ([_P, _P, _P], _I),
    "lt_global_split_begin": ([_P, _I, _I, _P], _I),
    "lt_global_split_step": ([_P, _P, _P, _P], _I),
    "lt_global_split_apply": ([_P, _P, _F, _F, _P], _I),
    "lt_global_split_result": ([_P, _P, _P], _I),
    "lt_get_bank": ([_P, _P, _P], _I),
    "lt_project": ([_P, _I, _P, _P, _P], _I),
    "lt_backproject": ([_P, _I, _P, _P, _P], _I),
    "lt_disc_correct": ([_P, _P, _P, _P, _P], _I),
    "lt_conv_cache": ([_P, _P, _P], _I),
    "lt_get_conv": ([_P, _P, _P], _I),
    "lt_sirt_solve": ([_P, _P, _F, _F, _P, _P], _I),
    "lt_tv_solve": ([_P, _P, _F, _I, _P, _P], _I),
    "lt_get_ext": ([_P, _P, _P], _I),
    "lt_combine_rois": ([_P, _P, _I, _P, _P, _P], _I),
    "lt_solve_host": ([_P, _I, _P, _F, _F, _I, _P, _P], _I),
    "lt_global_sirt": ([_P, _P, _I, _F, _F, _P, _P], _I),
    "lt_global_tv": ([_P, _P, _I, _F, _I, _P, _P], _I),
    "lt_fgp_batch": ([_I, _I, _I, _P, _F, _I, _P, _P], _I),
    "lt_pad_truncated": ([_P, _I, _I, _I, _P, _P], _I),
    "lt_tv_solve_lambdas": ([_P, _P, _P, _I, _P, _P], _I),
    "lt_haar_solve": ([_P, _P, _F, _I, _I, _P, _P], _I),
    "lt_global_cp": ([_P, _P, _I, _F, _P, _P], _I),
    "lt_exterior_solve": ([_P, _P, _F, _F, _P, _P], _I),
    "lt_combine_peers": ([_P, _P, _I, _I, _P, _P, _P], _I),
    "lt_ipc_get_handle": ([_P, _P], _I),
    "lt_ipc_open_handle": ([_P, _P], _I),
    "lt_ipc_close": ([_P], _I),
    "lt_metrics": ([_P, _P, _I, _I, _I, _F, _P, _P, _P], _I),
    "lt_nelder_mead_1d": ([_P, _P, ctypes.c_double, ctypes.c_double, _I, _P, _P, _P], _I),
    "lt_launch_count": ([], _i64),
    "lt_timing_enable": ([_I], None),
    "lt_timing_read": ([_P, _P], _I),
    "lt_plan_destroy": ([_P], None),
    "lt_last_error": ([], ctypes.c_char_p),
}
for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res

EXPORTS = tuple(_SIGS)


class LtError(RuntimeError):
    pass


def _chk(rc: int, what: str) -> None:
    if rc != LT_OK:
        msg = _lib.lt_last_error().decode()
        raise (ValueError if rc == LT_ERR_INVALID else LtError)(f"{what}: {msg} (code {rc})")


def _stream(dev=None) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _cuda_f32(t: torch.Tensor, name: str) -> torch.Tensor:
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32):
        raise TypeError(f"{name} must be a CUDA float32 tensor")
    return t.contiguous()


def launch_count() -> int:
    """Kernels launched by the library so far (process-wide)."""
    return int(_lib.lt_launch_count())


KERNEL_CLASSES = ("fp", "bp", "fgp", "conv", "xs")


def timing_enable(on: bool = True) -> None:
    """Bracket every FP/BP/FGP/conv launch with CUDA events on its stream."""
    _lib.lt_timing_enable(1 if on else 0)


def timing_read() -> dict:
    """{class: (total_ms, launches)} since the last read (synchronizes on the events)."""
    ms = np.zeros(len(KERNEL_CLASSES), dtype=np.float64)
    cnt = np.zeros(len(KERNEL_CLASSES), dtype=np.int64)
    _chk(_lib.lt_timing_read(ms.ctypes.data, cnt.ctypes.data), "lt_timing_read")
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_CLASSES)}


def window_width(h: int) -> int:
    return 2 * math.ceil((2 * h - 1) / math.sqrt(2) - 1e-12) + 4


class Plan:
    """One geometry + ROI batch (``lt_roi_setup``), with its device workspace.

    n, angles, n_det: grid size N, projection angles (rad), detector count N_d.
    centres: (R, 2) integer core centres (row, col); radius r, margin m.
    n_iter: outer iterations n (the filter bank holds u_1..u_n).
    """

    def __init__(self, n: int, angles, n_det: int, centres, radius: int, margin: int, n_iter: int,
                 disc: bool = True, rank: int = 0, world: int = 1, device=None, bind: bool = True,
                 xs_exact: bool = False):
        """bind=False plans on the host only (tables, partition); no device memory.
        xs_exact: x_s^k from the global SIRT iterate (LT_XS_EXACT, NEXT-4(i))."""
        if bind:
            self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        else:
            self.device = None
        ang = np.ascontiguousarray(np.asarray(angles, dtype=np.float64))
        cen = np.ascontiguousarray(np.asarray(centres, dtype=np.int32).reshape(-1, 2))
        rows = np.ascontiguousarray(cen[:, 0]); cols = np.ascontiguousarray(cen[:, 1])
        self.n, self.n_det, self.n_angles = int(n), int(n_det), len(ang)
        self.radius, self.margin, self.n_iter = int(radius), int(margin), int(n_iter)
        self.angles, self.centres = ang, cen
        self.h = self.radius + self.margin
        self._p = ctypes.c_void_p()
        _chk(_lib.lt_roi_setup(self.n, len(ang), self.n_det, ang.ctypes.data, len(cen), rows.ctypes.data,
                               cols.ctypes.data, self.radius, self.margin, self.n_iter,
                               (LT_DISC_ON if disc else 0) | (LT_XS_EXACT if xs_exact else 0), rank, world,
                               ctypes.byref(self._p)), "lt_roi_setup")
        self.workspace_bytes = nbytes = int(_lib.lt_plan_workspace_bytes(self._p))
        if bind:
            with torch.cuda.device(self.device):
                self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
                _chk(_lib.lt_plan_bind_workspace(self._p, self.ws.data_ptr(), nbytes, _stream(self.device)),
                     "lt_plan_bind_workspace")
        self.R = int(_lib.lt_plan_local_count(self._p))
        loc = np.zeros(max(self.R, 1), dtype=np.int32)
        _chk(_lib.lt_plan_local_rois(self._p, loc.ctypes.data), "lt_plan_local_rois")
        self.local_rois = loc[:self.R].copy()

    def __del__(self):
        p = getattr(self, "_p", None)
        if p is not None and p.value and _lib is not None:
            _lib.lt_plan_destroy(p)
            self._p = None

    def tables(self):
        """(rects [R, 6] = row0, col0, vr0, vr1, vc0, vc1; d0 [R, N_theta]; window width)."""
        R = max(self.R, 1)
        rects = np.zeros((R, 6), dtype=np.int32)
        d0 = np.zeros((R, self.n_angles), dtype=np.int32)
        w = ctypes.c_int32(0)
        _chk(_lib.lt_plan_tables(self._p, rects.ctypes.data, d0.ctypes.data, ctypes.byref(w)), "lt_plan_tables")
        return rects[:self.R], d0[:self.R], int(w.value)

    # ---- geometry / bank ---------------------------------------------------
    @property
    def alpha(self) -> float:
        return 1.0 / (self.n_angles * self.n_det)

    def _empty(self, *shape) -> torch.Tensor:
        return torch.empty(*shape, dtype=torch.float32, device=self.device)

    def filter_bank(self) -> None:
        _chk(_lib.lt_filter_bank(self._p, _stream(self.device)), "lt_filter_bank")

    def set_bank(self, bank: torch.Tensor) -> None:
        bank = _cuda_f32(bank, "bank")
        assert bank.numel() == self.n_iter * self.n_angles * self.n_det
        _chk(_lib.lt_set_bank(self._p, bank.data_ptr(), _stream(self.device)), "lt_set_bank")
        self._keep = bank

    # angle-split Alg. 1 (lt_bank_split_*; the all-reduce is the caller's, dist.filter_bank_split)
    def bank_split_begin(self, a0: int, a1: int) -> None:
        _chk(_lib.lt_bank_split_begin(self._p, a0, a1, _stream(self.device)), "lt_bank_split_begin")

    def bank_split_step(self, k: int, partial: torch.Tensor = None) -> None:
        ptr = None
        if partial is not None:
            assert partial.is_cuda and partial.dtype == torch.float32 and partial.is_contiguous()
            assert partial.numel() == self.n * self.n
            ptr = partial.data_ptr()
        _chk(_lib.lt_bank_split_step(self._p, k, ptr, _stream(self.device)), "lt_bank_split_step")

    def bank_split_apply(self, reduced: torch.Tensor) -> None:
        reduced = _cuda_f32(reduced, "reduced")
        assert reduced.numel() == self.n * self.n
        _chk(_lib.lt_bank_split_apply(self._p, reduced.data_ptr(), _stream(self.device)), "lt_bank_split_apply")

    # angle-split global box-SIRT (lt_global_split_*; dist.global_sirt_split)
    def global_split_begin(self, a0: int, a1: int) -> None:
        _chk(_lib.lt_global_split_begin(self._p, a0, a1, _stream(self.device)), "lt_global_split_begin")

    def global_split_step(self, sino: torch.Tensor, partial: torch.Tensor) -> None:
        sino = _cuda_f32(sino, "sino")
        assert partial.is_cuda and partial.dtype == torch.float32 and partial.is_contiguous()
        assert partial.numel() == self.n * self.n
        _chk(_lib.lt_global_split_step(self._p, sino.data_ptr(), partial.data_ptr(), _stream(self.device)),
             "lt_global_split_step")

    def global_split_apply(self, reduced: torch.Tensor, lo: float, hi: float) -> None:
        reduced = _cuda_f32(reduced, "reduced")
        assert reduced.numel() == self.n * self.n
        _chk(_lib.lt_global_split_apply(self._p, reduced.data_ptr(), float(lo), float(hi), _stream(self.device)),
             "lt_global_split_apply")

    def global_split_result(self) -> torch.Tensor:
        out = self._empty(self.n, self.n)
        _chk(_lib.lt_global_split_result(self._p, out.data_ptr(), _stream(self.device)), "lt_global_split_result")
        return out

    def get_bank(self) -> torch.Tensor:
        out = self._empty(self.n_iter, self.n_angles, self.n_det)
        _chk(_lib.lt_get_bank(self._p, out.data_ptr(), _stream(self.device)), "lt_get_bank")
        return out

    # ---- operators -----------------------------------------------------------
    def project(self, img: torch.Tensor, roi: int = -1) -> torch.Tensor:
        img = _cuda_f32(img, "img")
        out = self._empty(self.n_angles, self.n_det)
        _chk(_lib.lt_project(self._p, roi, img.data_ptr(), out.data_ptr(), _stream(self.device)), "lt_project")
        return out

    def backproject(self, sino: torch.Tensor, roi: int = -1) -> torch.Tensor:
        sino = _cuda_f32(sino, "sino")
        out = self._empty(self.n, self.n)
        _chk(_lib.lt_backproject(self._p, roi, sino.data_ptr(), out.data_ptr(), _stream(self.device)), "lt_backproject")
        return out

    def disc_correct(self, sino: torch.Tensor):
        sino = _cuda_f32(sino, "sino")
        pc = self._empty(self.n_angles, self.n_det)
        c = self._empty(1)
        _chk(_lib.lt_disc_correct(self._p, sino.data_ptr(), pc.data_ptr(), c.data_ptr(), _stream(self.device)),
             "lt_disc_correct")
        return pc, c

    def conv_cache(self, pc: torch.Tensor) -> torch.Tensor:
        pc = _cuda_f32(pc, "pc")
        _chk(_lib.lt_conv_cache(self._p, pc.data_ptr(), _stream(self.device)), "lt_conv_cache")
        out = self._empty(self.n_iter, self.n_angles, self.n_det)
        _chk(_lib.lt_get_conv(self._p, out.data_ptr(), _stream(self.device)), "lt_get_conv")
        return out

    # ---- solves ----------------------------------------------------------------
    def sirt_solve(self, sino: torch.Tensor, lo: float = 0.0, hi: float = math.inf,
                   out: Optional[torch.Tensor] = None) -> torch.Tensor:
        sino = _cuda_f32(sino, "sino")
        side = 2 * self.radius
        out = self._empty(self.R, side, side) if out is None else out
        _chk(_lib.lt_sirt_solve(self._p, sino.data_ptr(), lo, hi, out.data_ptr(), _stream(self.device)),
             "lt_sirt_solve")
        return out

    def tv_solve(self, sino: torch.Tensor, lam, n_fgp: int = 100,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """lam: one value, or one per local ROI (lambda sweep, lt_tv_solve_lambdas)."""
        sino = _cuda_f32(sino, "sino")
        side = 2 * self.radius
        out = self._empty(self.R, side, side) if out is None else out
        if np.ndim(lam) == 0:
            _chk(_lib.lt_tv_solve(self._p, sino.data_ptr(), float(lam), n_fgp, out.data_ptr(), _stream(self.device)),
                 "lt_tv_solve")
        else:
            lams = np.ascontiguousarray(np.asarray(lam, dtype=np.float32).reshape(-1))
            if lams.size != self.R:
                raise ValueError(f"{lams.size} lambdas for {self.R} local ROIs")
            _chk(_lib.lt_tv_solve_lambdas(self._p, sino.data_ptr(), lams.ctypes.data, n_fgp, out.data_ptr(),
                                          _stream(self.device)), "lt_tv_solve_lambdas")
        return out

    def exterior_solve(self, sino: torch.Tensor, lo: float = 0.0, hi: float = math.inf,
                       out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Exterior-subtraction ROI reconstruction (the prior art; lt_exterior_solve)."""
        sino = _cuda_f32(sino, "sino")
        side = 2 * self.radius
        out = self._empty(self.R, side, side) if out is None else out
        _chk(_lib.lt_exterior_solve(self._p, sino.data_ptr(), lo, hi, out.data_ptr(), _stream(self.device)),
             "lt_exterior_solve")
        return out

    def haar_solve(self, sino: torch.Tensor, lam: float, levels: int = 4, momentum: bool = True,
                   out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Local reconstruction with the Haar-wavelet l1 prior (lt_haar_solve)."""
        sino = _cuda_f32(sino, "sino")
        side = 2 * self.radius
        out = self._empty(self.R, side, side) if out is None else out
        _chk(_lib.lt_haar_solve(self._p, sino.data_ptr(), float(lam), int(levels), int(bool(momentum)),
                                out.data_ptr(), _stream(self.device)), "lt_haar_solve")
        return out

    def optimize_lambda(self, sino: torch.Tensor, ref_cores: torch.Tensor, target: str = "mse",
                        log10_bounds=(-3.0, 0.0), budget: int = 20, n_fgp: int = 100):
        """lambda minimising the mean MSE (or maximising the mean SSIM) of this
        plan's ROI cores against ref_cores by Nelder-Mead in log10(lambda)
        (PAPER.md L789-795): returns (lambda, value, evaluations)."""
        ref = _cuda_f32(ref_cores, "ref_cores")
        side = 2 * self.radius
        cores = self._empty(self.R, side, side)

        def objective(t):
            self.tv_solve(sino, 10.0 ** t, n_fgp, out=cores)
            mse, ssim = metrics(cores, ref)
            return float(mse.mean()) if target == "mse" else -float(ssim.mean())

        t, v, n = nelder_mead_1d(objective, log10_bounds[0], log10_bounds[1], budget)
        return 10.0 ** t, (v if target == "mse" else -v), n

    def get_ext(self) -> torch.Tensor:
        E = 2 * self.h
        out = self._empty(self.R, E, E)
        _chk(_lib.lt_get_ext(self._p, out.data_ptr(), _stream(self.device)), "lt_get_ext")
        return out

    def combine(self, cores_all: torch.Tensor, slot_roi: Sequence[int],
                out: Optional[torch.Tensor] = None) -> torch.Tensor:
        cores_all = _cuda_f32(cores_all, "cores_all")
        slots = np.ascontiguousarray(np.asarray(slot_roi, dtype=np.int32))
        out = self._empty(self.n, self.n) if out is None else out
        _chk(_lib.lt_combine_rois(self._p, cores_all.data_ptr(), len(slots), slots.ctypes.data, out.data_ptr(),
                                  _stream(self.device)), "lt_combine_rois")
        return out

    def combine_peers(self, peer_ptrs: Sequence[int], slots_per_rank: int, slot_roi: Sequence[int],
                      out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Combine reading every rank's [slots_per_rank, 2r, 2r] core buffer in place
        (device pointers valid in this process; lt_combine_peers)."""
        ptrs = (ctypes.c_void_p * len(peer_ptrs))(*[int(v) for v in peer_ptrs])
        slots = np.ascontiguousarray(np.asarray(slot_roi, dtype=np.int32))
        out = self._empty(self.n, self.n) if out is None else out
        _chk(_lib.lt_combine_peers(self._p, ptrs, len(peer_ptrs), int(slots_per_rank), slots.ctypes.data,
                                   out.data_ptr(), _stream(self.device)), "lt_combine_peers")
        return out

    def solve_host(self, mode: str, sino_host: torch.Tensor, p0: float, p1: float = 0.0, n_fgp: int = 100,
                   image_host: Optional[torch.Tensor] = None) -> torch.Tensor:
        """End-to-end with host buffers (pinned tensors recommended)."""
        assert not sino_host.is_cuda and sino_host.dtype == torch.float32 and sino_host.is_contiguous()
        if image_host is None:
            image_host = torch.empty(self.n, self.n, dtype=torch.float32, pin_memory=True)
        _chk(_lib.lt_solve_host(self._p, 0 if mode == "sirt" else 1, sino_host.data_ptr(), p0, p1, n_fgp,
                                image_host.data_ptr(), _stream(self.device)), "lt_solve_host")
        return image_host

    def global_sirt(self, sino: torch.Tensor, n_iter: int, lo: float = 0.0, hi: float = math.inf) -> torch.Tensor:
        sino = _cuda_f32(sino, "sino")
        out = self._empty(self.n, self.n)
        _chk(_lib.lt_global_sirt(self._p, sino.data_ptr(), n_iter, lo, hi, out.data_ptr(), _stream(self.device)),
             "lt_global_sirt")
        return out

    def global_cp(self, sino: torch.Tensor, n_iter: int, mu: float) -> torch.Tensor:
        """Chambolle-Pock TV (diagonal preconditioning) on the full grid (lt_global_cp)."""
        sino = _cuda_f32(sino, "sino")
        out = self._empty(self.n, self.n)
        _chk(_lib.lt_global_cp(self._p, sino.data_ptr(), n_iter, mu, out.data_ptr(), _stream(self.device)),
             "lt_global_cp")
        return out

    def global_tv(self, sino: torch.Tensor, n_iter: int, lam: float, n_fgp: int = 100) -> torch.Tensor:
        sino = _cuda_f32(sino, "sino")
        out = self._empty(self.n, self.n)
        _chk(_lib.lt_global_tv(self._p, sino.data_ptr(), n_iter, lam, n_fgp, out.data_ptr(), _stream(self.device)),
             "lt_global_tv")
        return out


def fgp_batch(x: torch.Tensor, lam: float, n_fgp: int) -> torch.Tensor:
    """FGP TV prox of each (h, w) image in x (count, h, w), the solver's kernel."""
    x = _cuda_f32(x, "x")
    cnt, h, w = x.shape
    out = torch.empty_like(x)
    _chk(_lib.lt_fgp_batch(h, w, cnt, x.data_ptr(), lam, n_fgp, out.data_ptr(), _stream(x.device)), "lt_fgp_batch")
    return out


def pad_truncated(sino_t: torch.Tensor, n_det: int, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Edge-constant, centred padding of truncated data ([N_theta, n_trunc] ->
    [N_theta, n_det]), PAPER.md L1134-1170 (lt_pad_truncated)."""
    sino_t = _cuda_f32(sino_t, "sino_t")
    na, nt = sino_t.shape
    if out is None:
        out = torch.empty(na, n_det, dtype=torch.float32, device=sino_t.device)
    out = _cuda_f32(out, "out")
    if tuple(out.shape) != (na, n_det):
        raise ValueError(f"out must be ({na}, {n_det})")
    _chk(_lib.lt_pad_truncated(sino_t.data_ptr(), na, nt, n_det, out.data_ptr(), _stream(sino_t.device)),
         "lt_pad_truncated")
    return out


def metrics(x: torch.Tensor, ref: torch.Tensor, data_range: Optional[float] = None):
    """(MSE, SSIM) per image of x vs ref ((count, h, w) or (h, w)), as float64
    CUDA tensors (lt_metrics)."""
    x = _cuda_f32(x, "x")
    ref = _cuda_f32(ref, "ref")
    if x.shape != ref.shape:
        raise ValueError("x and ref must have the same shape")
    x3 = x.reshape(-1, x.shape[-2], x.shape[-1])
    cnt, h, w = x3.shape
    mse = torch.empty(cnt, dtype=torch.float64, device=x.device)
    ssim = torch.empty(cnt, dtype=torch.float64, device=x.device)
    _chk(_lib.lt_metrics(x3.data_ptr(), ref.data_ptr(), cnt, h, w, float(data_range or 0.0), mse.data_ptr(),
                         ssim.data_ptr(), _stream(x.device)), "lt_metrics")
    return mse, ssim


_NM_CB = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_double, ctypes.c_void_p)


def nelder_mead_1d(f, t_lo: float, t_hi: float, budget: int):
    """Minimise f(t) over [t_lo, t_hi] with the library's 1-D Nelder-Mead
    (lt_nelder_mead_1d): returns (t_best, f_best, evaluations)."""
    err = []

    def cb(t, _ctx):
        try:
            return float(f(t))
        except Exception as e:   # noqa: BLE001 - re-raised after the C call returns
            err.append(e)
            return math.inf

    c = _NM_CB(cb)
    tb, fb, ne = ctypes.c_double(0.0), ctypes.c_double(0.0), ctypes.c_int32(0)
    _chk(_lib.lt_nelder_mead_1d(ctypes.cast(c, ctypes.c_void_p), None, t_lo, t_hi, budget, ctypes.byref(tb),
                                ctypes.byref(fb), ctypes.byref(ne)), "lt_nelder_mead_1d")
    if err:
        raise err[0]
    return tb.value, fb.value, ne.value


def ipc_handle(t: torch.Tensor) -> bytes:
    """64-byte CUDA IPC handle of the allocation holding t (lt_ipc_get_handle)."""
    buf = ctypes.create_string_buffer(64)
    _chk(_lib.lt_ipc_get_handle(t.data_ptr(), buf), "lt_ipc_get_handle")
    return buf.raw


def ipc_open(handle: bytes) -> int:
    """Device pointer of a peer's allocation in this process (lt_ipc_open_handle)."""
    ptr = ctypes.c_void_p(0)
    _chk(_lib.lt_ipc_open_handle(ctypes.create_string_buffer(handle, 64), ctypes.byref(ptr)), "lt_ipc_open_handle")
    return int(ptr.value)


def ipc_close(ptr: int) -> None:
    _chk(_lib.lt_ipc_close(ctypes.c_void_p(ptr)), "lt_ipc_close")
