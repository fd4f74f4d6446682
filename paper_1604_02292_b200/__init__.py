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
if os.environ.get("LT_SO"):          # diagnostics only (tools/ab.sh): an alternative build of the same library
    LIB_PATH = os.environ["LT_SO"]

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the CUDA extension is required; there is no fallback)")

_lib = ctypes.CDLL(LIB_PATH)

LT_OK, LT_ERR_RUNTIME, LT_ERR_INVALID = 0, 1, 2
LT_DISC_ON = 1
LT_XS_EXACT = 2
LT_GUARD_BANDS = 4

_P = ctypes.c_void_p
_I = ctypes.c_int32
_F = ctypes.c_float
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64

_SIGS = {
    "lt_roi_setup": ([_I, _I, _I, _P, _I, _P, _P, _I, _I, _I, _I, _I, _I, _P], _I),
    "lt_plan_workspace_bytes": ([_P], _i64),
    "lt_plan_bind_workspace": ([_P, _P, _i64, _P], _I),
    "lt_plan_local_count": ([_P], _I),
    "lt_plan_local_rois": ([_P, _P], _I),
    "lt_plan_tables": ([_P, _P, _P, _P], _I),
    "lt_filter_bank": ([_P, _P], _I),
    "lt_set_bank": ([_P, _P, _u64, _P], _I),
    "lt_bank_key": ([_P], _u64),
    "lt_save_bank": ([_P, ctypes.c_char_p, _P], _I),
    "lt_load_bank": ([_P, ctypes.c_char_p, _P], _I),
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
    "lt_combine_rois": ([_P, _P, _P, _P, _P], _I),
    "lt_stitch_slots": ([_P, _P, _I, _P, _P, _P], _I),
    "lt_plan_slot_table": ([_P, _P, _P], _I),
    "lt_nccl_get_unique_id": ([_P], _I),
    "lt_nccl_comm_init": ([_I, _I, _P, _P], _I),
    "lt_nccl_comm_destroy": ([_P], _I),
    "lt_window_width": ([_I], _I),
    "lt_guard_check": ([_P, _P, _P, _P], _I),
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


def _cuda_f32(t: torch.Tensor, name: str, device=None) -> torch.Tensor:
    """An input: a CUDA float32 tensor (on `device` when given), made contiguous."""
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32):
        raise TypeError(f"{name} must be a CUDA float32 tensor")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, the plan on {device}")
    return t.contiguous()


def _out_f32(t: Optional[torch.Tensor], shape, device, name: str = "out") -> torch.Tensor:
    """An output buffer: allocated when None, else it must be a contiguous CUDA
    float32 tensor of exactly `shape` on `device` (the library writes
    prod(shape) floats from its data pointer)."""
    shape = tuple(int(v) for v in shape)
    if t is None:
        return torch.empty(shape, dtype=torch.float32, device=device)
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32):
        raise TypeError(f"{name} must be a CUDA float32 tensor")
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if tuple(t.shape) != shape:
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {shape}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


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
    """The library's detector window width W(h) of an extended half-side h (lt_window_width)."""
    w = int(_lib.lt_window_width(int(h)))
    if w < 0:
        raise ValueError("h must be >= 1")
    return w


class Plan:
    """One geometry + ROI batch (``lt_roi_setup``), with its device workspace.

    n, angles, n_det: grid size N, projection angles (rad), detector count N_d.
    centres: (R, 2) integer core centres (row, col); radius r, margin m.
    n_iter: outer iterations n (the filter bank holds u_1..u_n).
    """

    def __init__(self, n: int, angles, n_det: int, centres, radius: int, margin: int, n_iter: int,
                 disc: bool = True, rank: int = 0, world: int = 1, device=None, bind: bool = True,
                 xs_exact: bool = False, guard_bands: bool = False):
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
        self.rank, self.world = int(rank), int(world)
        self._p = ctypes.c_void_p()
        _chk(_lib.lt_roi_setup(self.n, len(ang), self.n_det, ang.ctypes.data, len(cen), rows.ctypes.data,
                               cols.ctypes.data, self.radius, self.margin, self.n_iter,
                               (LT_DISC_ON if disc else 0) | (LT_XS_EXACT if xs_exact else 0)
                               | (LT_GUARD_BANDS if guard_bands else 0), rank, world,
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

    # ---- device plumbing ----------------------------------------------------
    def _dev(self):
        """Every library call runs with the plan's device current, so launches
        (and the legacy-stream handle 0) go to the GPU that holds the workspace."""
        if self.device is None:
            raise ValueError("plan is not bound to a device (bind=False)")
        return torch.cuda.device(self.device)

    def _st(self) -> int:
        return _stream(self.device)

    def _in(self, t: torch.Tensor, name: str, numel: Optional[int] = None) -> torch.Tensor:
        t = _cuda_f32(t, name, self.device)
        if numel is not None and t.numel() != numel:
            raise ValueError(f"{name} has {t.numel()} elements, expected {numel}")
        return t

    def _out(self, t: Optional[torch.Tensor], *shape) -> torch.Tensor:
        return _out_f32(t, shape, self.device)

    # ---- geometry / bank ---------------------------------------------------
    @property
    def alpha(self) -> float:
        return 1.0 / (self.n_angles * self.n_det)

    @property
    def bank_key(self) -> int:
        """64-bit key of the geometry the filters depend on (lt_bank_key)."""
        return int(_lib.lt_bank_key(self._p))

    def guard_check(self):
        """(damaged canary bands, first damaged workspace offset or -1) of a
        guard_bands=True plan (lt_guard_check; synchronizes the stream)."""
        off = ctypes.c_int64(-1)
        bad = ctypes.c_int32(0)
        with self._dev():
            _chk(_lib.lt_guard_check(self._p, ctypes.byref(bad), ctypes.byref(off), self._st()), "lt_guard_check")
        return int(bad.value), int(off.value)

    def slot_table(self):
        """(slots_per_rank, slot -> global ROI table [world * spr]) of the partition (lt_plan_slot_table)."""
        spr = ctypes.c_int32(0)
        _chk(_lib.lt_plan_slot_table(self._p, None, ctypes.byref(spr)), "lt_plan_slot_table")
        tab = np.zeros(self.world * spr.value, dtype=np.int32)
        _chk(_lib.lt_plan_slot_table(self._p, tab.ctypes.data, None), "lt_plan_slot_table")
        return spr.value, tab

    def filter_bank(self) -> None:
        with self._dev():
            _chk(_lib.lt_filter_bank(self._p, self._st()), "lt_filter_bank")

    def set_bank(self, bank: torch.Tensor, key: Optional[int] = None) -> None:
        """Install a bank [n_iter, N_theta, N_d] computed for the geometry with
        `key` (default: this plan's own key, i.e. the caller vouches for it)."""
        bank = self._in(bank, "bank", self.n_iter * self.n_angles * self.n_det)
        with self._dev():
            _chk(_lib.lt_set_bank(self._p, bank.data_ptr(), self.bank_key if key is None else int(key), self._st()),
                 "lt_set_bank")
        self._keep = bank

    def save_bank(self, path: str) -> None:
        with self._dev():
            _chk(_lib.lt_save_bank(self._p, os.fsencode(path), self._st()), "lt_save_bank")

    def load_bank(self, path: str) -> None:
        with self._dev():
            _chk(_lib.lt_load_bank(self._p, os.fsencode(path), self._st()), "lt_load_bank")

    # angle-split Alg. 1 (lt_bank_split_*; the all-reduce is the caller's, dist.filter_bank_split)
    def bank_split_begin(self, a0: int, a1: int) -> None:
        with self._dev():
            _chk(_lib.lt_bank_split_begin(self._p, a0, a1, self._st()), "lt_bank_split_begin")

    def bank_split_step(self, k: int, partial: torch.Tensor = None) -> None:
        ptr = None
        if partial is not None:
            partial = _out_f32(partial, tuple(partial.shape), self.device, "partial")
            if partial.numel() != self.n * self.n:
                raise ValueError("partial must hold N x N floats")
            ptr = partial.data_ptr()
        with self._dev():
            _chk(_lib.lt_bank_split_step(self._p, k, ptr, self._st()), "lt_bank_split_step")

    def bank_split_apply(self, reduced: torch.Tensor) -> None:
        reduced = self._in(reduced, "reduced", self.n * self.n)
        with self._dev():
            _chk(_lib.lt_bank_split_apply(self._p, reduced.data_ptr(), self._st()), "lt_bank_split_apply")

    # angle-split global box-SIRT (lt_global_split_*; dist.global_sirt_split)
    def global_split_begin(self, a0: int, a1: int) -> None:
        with self._dev():
            _chk(_lib.lt_global_split_begin(self._p, a0, a1, self._st()), "lt_global_split_begin")

    def global_split_step(self, sino: torch.Tensor, partial: torch.Tensor) -> None:
        sino = self._in(sino, "sino", self.n_angles * self.n_det)
        partial = _out_f32(partial, tuple(partial.shape), self.device, "partial")
        if partial.numel() != self.n * self.n:
            raise ValueError("partial must hold N x N floats")
        with self._dev():
            _chk(_lib.lt_global_split_step(self._p, sino.data_ptr(), partial.data_ptr(), self._st()),
                 "lt_global_split_step")

    def global_split_apply(self, reduced: torch.Tensor, lo: float, hi: float) -> None:
        reduced = self._in(reduced, "reduced", self.n * self.n)
        with self._dev():
            _chk(_lib.lt_global_split_apply(self._p, reduced.data_ptr(), float(lo), float(hi), self._st()),
                 "lt_global_split_apply")

    def global_split_result(self) -> torch.Tensor:
        out = self._out(None, self.n, self.n)
        with self._dev():
            _chk(_lib.lt_global_split_result(self._p, out.data_ptr(), self._st()), "lt_global_split_result")
        return out

    def get_bank(self) -> torch.Tensor:
        out = self._out(None, self.n_iter, self.n_angles, self.n_det)
        with self._dev():
            _chk(_lib.lt_get_bank(self._p, out.data_ptr(), self._st()), "lt_get_bank")
        return out

    # ---- operators -----------------------------------------------------------
    def project(self, img: torch.Tensor, roi: int = -1) -> torch.Tensor:
        img = self._in(img, "img", self.n * self.n)
        out = self._out(None, self.n_angles, self.n_det)
        with self._dev():
            _chk(_lib.lt_project(self._p, roi, img.data_ptr(), out.data_ptr(), self._st()), "lt_project")
        return out

    def backproject(self, sino: torch.Tensor, roi: int = -1) -> torch.Tensor:
        sino = self._in(sino, "sino", self.n_angles * self.n_det)
        out = self._out(None, self.n, self.n)
        with self._dev():
            _chk(_lib.lt_backproject(self._p, roi, sino.data_ptr(), out.data_ptr(), self._st()), "lt_backproject")
        return out

    def disc_correct(self, sino: torch.Tensor):
        sino = self._in(sino, "sino", self.n_angles * self.n_det)
        pc = self._out(None, self.n_angles, self.n_det)
        c = self._out(None, 1)
        with self._dev():
            _chk(_lib.lt_disc_correct(self._p, sino.data_ptr(), pc.data_ptr(), c.data_ptr(), self._st()),
                 "lt_disc_correct")
        return pc, c

    def conv_cache(self, pc: torch.Tensor) -> torch.Tensor:
        pc = self._in(pc, "pc", self.n_angles * self.n_det)
        out = self._out(None, self.n_iter, self.n_angles, self.n_det)
        with self._dev():
            _chk(_lib.lt_conv_cache(self._p, pc.data_ptr(), self._st()), "lt_conv_cache")
            _chk(_lib.lt_get_conv(self._p, out.data_ptr(), self._st()), "lt_get_conv")
        return out

    # ---- solves ----------------------------------------------------------------
    def _cores_out(self, out):
        side = 2 * self.radius
        return self._out(out, self.R, side, side)

    def sirt_solve(self, sino: torch.Tensor, lo: float = 0.0, hi: float = math.inf,
                   out: Optional[torch.Tensor] = None) -> torch.Tensor:
        sino = self._in(sino, "sino", self.n_angles * self.n_det)
        out = self._cores_out(out)
        with self._dev():
            _chk(_lib.lt_sirt_solve(self._p, sino.data_ptr(), lo, hi, out.data_ptr(), self._st()), "lt_sirt_solve")
        return out

    def tv_solve(self, sino: torch.Tensor, lam, n_fgp: int = 100,
                 out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """lam: one value, or one per local ROI (lambda sweep, lt_tv_solve_lambdas)."""
        sino = self._in(sino, "sino", self.n_angles * self.n_det)
        out = self._cores_out(out)
        with self._dev():
            if np.ndim(lam) == 0:
                _chk(_lib.lt_tv_solve(self._p, sino.data_ptr(), float(lam), n_fgp, out.data_ptr(), self._st()),
                     "lt_tv_solve")
            else:
                lams = np.ascontiguousarray(np.asarray(lam, dtype=np.float32).reshape(-1))
                if lams.size != self.R:
                    raise ValueError(f"{lams.size} lambdas for {self.R} local ROIs")
                _chk(_lib.lt_tv_solve_lambdas(self._p, sino.data_ptr(), lams.ctypes.data, n_fgp, out.data_ptr(),
                                              self._st()), "lt_tv_solve_lambdas")
        return out

    def exterior_solve(self, sino: torch.Tensor, lo: float = 0.0, hi: float = math.inf,
                       out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Exterior-subtraction ROI reconstruction (the prior art; lt_exterior_solve)."""
        sino = self._in(sino, "sino", self.n_angles * self.n_det)
        out = self._cores_out(out)
        with self._dev():
            _chk(_lib.lt_exterior_solve(self._p, sino.data_ptr(), lo, hi, out.data_ptr(), self._st()),
                 "lt_exterior_solve")
        return out

    def haar_solve(self, sino: torch.Tensor, lam: float, levels: int = 4, momentum: bool = True,
                   out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Local reconstruction with the Haar-wavelet l1 prior (lt_haar_solve)."""
        sino = self._in(sino, "sino", self.n_angles * self.n_det)
        out = self._cores_out(out)
        with self._dev():
            _chk(_lib.lt_haar_solve(self._p, sino.data_ptr(), float(lam), int(levels), int(bool(momentum)),
                                    out.data_ptr(), self._st()), "lt_haar_solve")
        return out

    def optimize_lambda(self, sino: torch.Tensor, ref_cores: torch.Tensor, target: str = "mse",
                        log10_bounds=(-3.0, 0.0), budget: int = 20, n_fgp: int = 100):
        """lambda minimising the mean MSE (or maximising the mean SSIM) of this
        plan's ROI cores against ref_cores by Nelder-Mead in log10(lambda)
        (PAPER.md L789-795): returns (lambda, value, evaluations)."""
        ref = self._in(ref_cores, "ref_cores")
        cores = self._cores_out(None)

        def objective(t):
            self.tv_solve(sino, 10.0 ** t, n_fgp, out=cores)
            mse, ssim = metrics(cores, ref)
            return float(mse.mean()) if target == "mse" else -float(ssim.mean())

        t, v, n = nelder_mead_1d(objective, log10_bounds[0], log10_bounds[1], budget)
        return 10.0 ** t, (v if target == "mse" else -v), n

    def get_ext(self) -> torch.Tensor:
        E = 2 * self.h
        out = self._out(None, self.R, E, E)
        with self._dev():
            _chk(_lib.lt_get_ext(self._p, out.data_ptr(), self._st()), "lt_get_ext")
        return out

    def combine(self, cores_all: torch.Tensor, slot_roi: Sequence[int],
                out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Stitch already-gathered cores [n_slots, 2r, 2r] (lt_stitch_slots)."""
        slots = np.ascontiguousarray(np.asarray(slot_roi, dtype=np.int32))
        side = 2 * self.radius
        cores_all = self._in(cores_all, "cores_all", len(slots) * side * side)
        out = self._out(out, self.n, self.n)
        with self._dev():
            _chk(_lib.lt_stitch_slots(self._p, cores_all.data_ptr(), len(slots), slots.ctypes.data, out.data_ptr(),
                                      self._st()), "lt_stitch_slots")
        return out

    def combine_rois(self, cores: torch.Tensor, comm: Optional["NcclComm"] = None,
                     out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """The full image on every rank from this rank's cores (lt_combine_rois:
        library-owned NCCL all-gather + stitch; comm may be None on one rank)."""
        side = 2 * self.radius
        cores = self._in(cores, "cores", self.R * side * side)
        out = self._out(out, self.n, self.n)
        with self._dev():
            _chk(_lib.lt_combine_rois(self._p, cores.data_ptr(), out.data_ptr(), comm.handle if comm else None,
                                      self._st()), "lt_combine_rois")
        return out

    def combine_peers(self, peer_ptrs: Sequence[int], slots_per_rank: int, slot_roi: Sequence[int],
                      out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Combine reading every rank's [slots_per_rank, 2r, 2r] core buffer in place
        (device pointers valid in this process; lt_combine_peers)."""
        ptrs = (ctypes.c_void_p * len(peer_ptrs))(*[int(v) for v in peer_ptrs])
        slots = np.ascontiguousarray(np.asarray(slot_roi, dtype=np.int32))
        out = self._out(out, self.n, self.n)
        with self._dev():
            _chk(_lib.lt_combine_peers(self._p, ptrs, len(peer_ptrs), int(slots_per_rank), slots.ctypes.data,
                                       out.data_ptr(), self._st()), "lt_combine_peers")
        return out

    def solve_host(self, mode: str, sino_host: torch.Tensor, p0: float, p1: float = 0.0, n_fgp: int = 100,
                   image_host: Optional[torch.Tensor] = None) -> torch.Tensor:
        """End-to-end with host buffers (pinned tensors recommended)."""
        if not (isinstance(sino_host, torch.Tensor) and not sino_host.is_cuda and sino_host.dtype == torch.float32
                and sino_host.is_contiguous() and sino_host.numel() == self.n_angles * self.n_det):
            raise ValueError("sino_host must be a contiguous CPU float32 tensor of N_theta x N_d")
        if image_host is None:
            image_host = torch.empty(self.n, self.n, dtype=torch.float32, pin_memory=True)
        if not (isinstance(image_host, torch.Tensor) and not image_host.is_cuda
                and image_host.dtype == torch.float32 and image_host.is_contiguous()
                and image_host.numel() == self.n * self.n):
            raise ValueError("image_host must be a contiguous CPU float32 tensor of N x N")
        if mode not in ("sirt", "tv"):
            raise ValueError("mode must be 'sirt' or 'tv'")
        with self._dev():
            _chk(_lib.lt_solve_host(self._p, 0 if mode == "sirt" else 1, sino_host.data_ptr(), p0, p1, n_fgp,
                                    image_host.data_ptr(), self._st()), "lt_solve_host")
        return image_host

    def global_sirt(self, sino: torch.Tensor, n_iter: int, lo: float = 0.0, hi: float = math.inf) -> torch.Tensor:
        sino = self._in(sino, "sino", self.n_angles * self.n_det)
        out = self._out(None, self.n, self.n)
        with self._dev():
            _chk(_lib.lt_global_sirt(self._p, sino.data_ptr(), n_iter, lo, hi, out.data_ptr(), self._st()),
                 "lt_global_sirt")
        return out

    def global_cp(self, sino: torch.Tensor, n_iter: int, mu: float) -> torch.Tensor:
        """Chambolle-Pock TV (diagonal preconditioning) on the full grid (lt_global_cp)."""
        sino = self._in(sino, "sino", self.n_angles * self.n_det)
        out = self._out(None, self.n, self.n)
        with self._dev():
            _chk(_lib.lt_global_cp(self._p, sino.data_ptr(), n_iter, mu, out.data_ptr(), self._st()), "lt_global_cp")
        return out

    def global_tv(self, sino: torch.Tensor, n_iter: int, lam: float, n_fgp: int = 100) -> torch.Tensor:
        sino = self._in(sino, "sino", self.n_angles * self.n_det)
        out = self._out(None, self.n, self.n)
        with self._dev():
            _chk(_lib.lt_global_tv(self._p, sino.data_ptr(), n_iter, lam, n_fgp, out.data_ptr(), self._st()),
                 "lt_global_tv")
        return out


class NcclComm:
    """The library's NCCL communicator for lt_combine_rois:
    rank 0 creates the unique id (lt_nccl_get_unique_id), torch.distributed
    broadcasts its 128 bytes, every rank calls ncclCommInitRank through
    lt_nccl_comm_init on its current device."""

    def __init__(self, world: int, rank: int, unique_id: bytes, device=None):
        self.world, self.rank = int(world), int(rank)
        self.handle = None
        h = ctypes.c_void_p()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        with torch.cuda.device(dev):
            _chk(_lib.lt_nccl_comm_init(self.world, self.rank, ctypes.create_string_buffer(bytes(unique_id), 128),
                                        ctypes.byref(h)), "lt_nccl_comm_init")
        self.handle = h.value

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _chk(_lib.lt_nccl_get_unique_id(buf), "lt_nccl_get_unique_id")
        return buf.raw

    @classmethod
    def from_process_group(cls, group=None, device=None) -> "NcclComm":
        """Exchange the id over torch.distributed (rank 0 -> all) and init."""
        import torch.distributed as dist
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = cls.unique_id() if rank == 0 else bytes(128)
        if world > 1:
            dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
            t = torch.tensor(list(uid), dtype=torch.uint8,
                             device=dev if dist.get_backend(group) == "nccl" else "cpu")
            dist.broadcast(t, 0, group=group)
            uid = bytes(t.cpu().tolist())
        return cls(world, rank, uid, device)

    def close(self) -> None:
        if self.handle:
            _chk(_lib.lt_nccl_comm_destroy(ctypes.c_void_p(self.handle)), "lt_nccl_comm_destroy")
            self.handle = None


def fgp_batch(x: torch.Tensor, lam: float, n_fgp: int) -> torch.Tensor:
    """FGP TV prox of each (h, w) image in x (count, h, w), the solver's kernel."""
    x = _cuda_f32(x, "x")
    if x.dim() != 3:
        raise ValueError("x must be (count, h, w)")
    cnt, h, w = x.shape
    out = torch.empty_like(x)
    with torch.cuda.device(x.device):
        _chk(_lib.lt_fgp_batch(h, w, cnt, x.data_ptr(), lam, n_fgp, out.data_ptr(), _stream(x.device)),
             "lt_fgp_batch")
    return out


def pad_truncated(sino_t: torch.Tensor, n_det: int, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Edge-constant, centred padding of truncated data ([N_theta, n_trunc] ->
    [N_theta, n_det]), PAPER.md L1134-1170 (lt_pad_truncated)."""
    sino_t = _cuda_f32(sino_t, "sino_t")
    na, nt = sino_t.shape
    out = _out_f32(out, (na, n_det), sino_t.device)
    with torch.cuda.device(sino_t.device):
        _chk(_lib.lt_pad_truncated(sino_t.data_ptr(), na, nt, n_det, out.data_ptr(), _stream(sino_t.device)),
             "lt_pad_truncated")
    return out


def metrics(x: torch.Tensor, ref: torch.Tensor, data_range: Optional[float] = None):
    """(MSE, SSIM) per image of x vs ref ((count, h, w) or (h, w)), as float64
    CUDA tensors (lt_metrics)."""
    x = _cuda_f32(x, "x")
    ref = _cuda_f32(ref, "ref", x.device)
    if x.shape != ref.shape:
        raise ValueError("x and ref must have the same shape")
    x3 = x.reshape(-1, x.shape[-2], x.shape[-1])
    cnt, h, w = x3.shape
    mse = torch.empty(cnt, dtype=torch.float64, device=x.device)
    ssim = torch.empty(cnt, dtype=torch.float64, device=x.device)
    with torch.cuda.device(x.device):
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
