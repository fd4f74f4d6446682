"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no W, no W^T, no filters,
no solvers).  It only produces inputs:

* random phantoms of additive ellipses / rotated rectangles shaped like the
  paper's piecewise-constant, sparse-boundary objects;
* their sinograms as *analytic* line integrals, averaged over 4 sub-rays per
  detector bin (the intent of the paper's 4x detector supersampling,
  PAPER.md L800-804, without the inverse crime);
* the paper's noise models: Poisson with peak count I0 (PAPER.md L805-812,
  reading A16 in DESIGN.md) and Gaussian (BASELINE.json configs);
* ROI centre lists (seeded positions or tilings, BASELINE.json configs).

Seeds: ``np.random.default_rng([cfg_id, stream])`` with stream 0 = phantom,
1 = noise, 2 = ROI positions.

Geometry convention (V1 in DESIGN.md): pixel (i, j) has centre
x_j = j - (N-1)/2, y_i = (N-1)/2 - i; detector bin d has centre
t_d = d - (N_d-1)/2; the ray of angle theta at t is {x cos + y sin = t}.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "Shape", "Config", "CONFIGS", "config", "angles_for", "random_shapes",
    "analytic_sinogram", "raster", "add_noise", "roi_centres", "make_inputs",
    "seeded_rng", "sweep_lambdas",
]


def seeded_rng(cfg_id: int, stream: int) -> np.random.Generator:
    return np.random.default_rng([int(cfg_id), int(stream)])


@dataclasses.dataclass(frozen=True)
class Shape:
    kind: str          # "ellipse" or "rect"
    x0: float
    y0: float
    a: float           # semi-axis / half-side along the rotated x axis
    b: float           # semi-axis / half-side along the rotated y axis
    phi: float         # rotation (rad)
    rho: float         # additive density


@dataclasses.dataclass(frozen=True)
class Config:
    cfg_id: int
    name: str
    n: int             # image N (N x N)
    n_angles: int
    span: float        # angles uniform in [0, span)
    n_det: int
    noise: str         # "gauss" or "poisson"
    noise_level: float # sigma fraction of max(p) or I0
    n_roi: int
    radius: int        # half-side r of the square core
    margin: int        # m; extended half-side h = r + m
    layout: str        # "centre", "seeded" or "tiling"
    n_iter: int
    solver: str        # "sirt", "tv" or "sirt+tv"
    lam: float
    n_fgp: int
    n_ellipses: int
    n_rects: int
    n_trunc: int = 0   # > 0: only the central n_trunc detector bins are measured


# BASELINE.json "configs", in order (C1..C5).  lambda for C3/C4 is not given
# by the config text; 0.05 (the C2 value) is used and stated in DESIGN.md.
CONFIGS = {
    "C1": Config(1, "C1", 64, 32, math.pi, 91, "gauss", 0.01, 1, 12, 8,
                 "centre", 100, "sirt", 0.0, 100, 5, 0),
    "C2": Config(2, "C2", 512, 64, math.pi, 725, "poisson", 1e4, 16, 32, 32,
                 "seeded", 200, "tv", 0.05, 100, 16, 0),
    "C3": Config(3, "C3", 1024, 32, 2.0 * math.pi / 3.0, 1449, "gauss", 0.02,
                 64, 48, 48, "seeded", 300, "sirt+tv", 0.05, 100, 25, 25),
    "C4": Config(4, "C4", 2048, 180, math.pi, 2897, "poisson", 5e3, 256, 64,
                 64, "tiling", 200, "tv", 0.05, 100, 32, 0),
    "C5": Config(5, "C5", 4096, 256, math.pi, 5793, "gauss", 0.01, 1024, 64,
                 64, "tiling", 500, "sirt", 0.0, 100, 64, 0),
    # SURVEY §8(f) NEXT-3, the paper's truncated-data experiment (PAPER.md L1143-1148:
    # 1024 detectors truncated to the central 256, 512 angles on [0, pi), Poisson
    # noise, TV, central ROI): here N = 1024 with the full detector N_d = 1449
    # truncated to the central 257 bins (odd, so it stays centred), I0 = 1e4 (the
    # paper gives none for this figure), a central 192^2 core with margin 32
    # (extended side 256, the kernels' maximum).
    "T1": Config(6, "T1", 1024, 512, math.pi, 1449, "poisson", 1e4, 1, 96, 32,
                 "centre", 200, "tv", 0.05, 100, 25, 0, 257),
    # SURVEY §8(f) NEXT-1, the lambda-sweep / parameter-estimation workload
    # (PAPER.md L789-795, L1116-1120): C2's geometry and noise, 4 seeded ROIs
    # each solved for 16 lambdas log-spaced in [1e-3, 1] in one batch (64
    # ROI-lambda solves), scored by MSE and SSIM against the ground truth.
    "L1": Config(7, "L1", 512, 64, math.pi, 725, "poisson", 1e4, 64, 32, 32,
                 "sweep", 200, "tv", 0.05, 100, 16, 0),
    # The paper's own local-part experiment (PAPER.md L845-849, L874-875,
    # L796-798): 1024^2 grid, 1024 detector pixels (1025: odd, reading A3; the
    # phantom lies inside the inscribed disc, so no data are truncated), 512
    # angles on [0, pi), Poisson noise (I0 = 1e4: the paper varies it), one
    # central 256^2 local part padded by 1/8 of its size on each side
    # (margin 32, extended side 320), FISTA-TV, 200 x 100 FGP
    # iterations; piecewise-constant ellipses and rectangles stand in for the
    # motor phantom (not distributed).
    "P1": Config(8, "P1", 1024, 512, math.pi, 1025, "poisson", 1e4, 1, 128, 32,
                 "centre", 200, "tv", 0.05, 100, 25, 25),
}

SWEEP_ROIS, SWEEP_LAMBDAS = 4, 16


def sweep_lambdas(cfg: "Config") -> np.ndarray:
    """Per-ROI lambda of a "sweep" layout: 16 values log-spaced in [1e-3, 1],
    repeated for each of the 4 ROI positions (ROI-major)."""
    return np.tile(np.logspace(-3.0, 0.0, SWEEP_LAMBDAS), cfg.n_roi // SWEEP_LAMBDAS)


def config(name: str) -> Config:
    return CONFIGS[name]


def angles_for(n_angles: int, span: float = math.pi) -> np.ndarray:
    """theta_a = a * span / N_theta, a = 0..N_theta-1 (fp64, strictly increasing)."""
    return np.arange(n_angles, dtype=np.float64) * (span / n_angles)


def random_shapes(n: int, n_ellipses: int, n_rects: int, rng: np.random.Generator) -> List[Shape]:
    """Additive shapes: rho ~ U[0,1], phi ~ U[0,pi), semi-axes ~ U[0.03N, 0.2N]
    (rect half-sides ~ U[0.02N, 0.12N]); centres uniform in the disc of radius
    0.4N - max axis so every object stays inside the inscribed circle.
    Ellipses and rectangles alternate when both are requested."""
    kinds: List[str] = []
    ne, nr = n_ellipses, n_rects
    while ne or nr:
        if ne:
            kinds.append("ellipse"); ne -= 1
        if nr:
            kinds.append("rect"); nr -= 1
    shapes = []
    for kind in kinds:
        if kind == "ellipse":
            a, b = rng.uniform(0.03 * n, 0.2 * n, size=2)
        else:
            a, b = rng.uniform(0.02 * n, 0.12 * n, size=2)
        phi = rng.uniform(0.0, math.pi)
        rho = rng.uniform(0.0, 1.0)
        reach = math.hypot(a, b) if kind == "rect" else max(a, b)
        rmax = max(0.0, 0.4 * n - reach)
        rr = rmax * math.sqrt(rng.uniform(0.0, 1.0))
        ang = rng.uniform(0.0, 2.0 * math.pi)
        shapes.append(Shape(kind, rr * math.cos(ang), rr * math.sin(ang), float(a), float(b),
                            float(phi), float(rho)))
    return shapes


def _chord_ellipse(s: Shape, theta: np.ndarray, t: np.ndarray) -> np.ndarray:
    """Line integral of a uniform ellipse over {x cos + y sin = t}:
    2 rho a b sqrt(a_t^2 - t'^2) / a_t^2 with a_t^2 = a^2 cos^2(theta-phi)
    + b^2 sin^2(theta-phi), t' = t - (x0 cos + y0 sin)  (Kak & Slaney)."""
    c, sn = np.cos(theta), np.sin(theta)
    at2 = (s.a * np.cos(theta - s.phi)) ** 2 + (s.b * np.sin(theta - s.phi)) ** 2
    tp = t - (s.x0 * c + s.y0 * sn)
    arg = at2 - tp * tp
    out = np.where(arg > 0.0, 2.0 * s.rho * s.a * s.b * np.sqrt(np.maximum(arg, 0.0)) / at2, 0.0)
    return out


def _chord_rect(s: Shape, theta: np.ndarray, t: np.ndarray) -> np.ndarray:
    """Length of {x cos + y sin = t} inside a rotated rectangle (slab clipping), times rho."""
    c, sn = np.cos(theta), np.sin(theta)
    # point on the line and its direction, in the rectangle frame
    px = t * c - s.x0
    py = t * sn - s.y0
    dx, dy = -sn, c
    cp, sp = math.cos(s.phi), math.sin(s.phi)
    qx = px * cp + py * sp
    qy = -px * sp + py * cp
    ex = dx * cp + dy * sp
    ey = -dx * sp + dy * cp
    lo = np.full(np.broadcast(qx, ex).shape, -np.inf)
    hi = np.full_like(lo, np.inf)
    for q, e, half in ((qx, ex, s.a), (qy, ey, s.b)):
        q = np.broadcast_to(q, lo.shape)
        e = np.broadcast_to(e, lo.shape)
        small = np.abs(e) < 1e-15
        with np.errstate(divide="ignore", invalid="ignore"):
            s1 = (-half - q) / e
            s2 = (half - q) / e
        smin = np.where(small, np.where(np.abs(q) <= half, -np.inf, np.inf), np.minimum(s1, s2))
        smax = np.where(small, np.where(np.abs(q) <= half, np.inf, -np.inf), np.maximum(s1, s2))
        lo = np.maximum(lo, smin)
        hi = np.minimum(hi, smax)
    return s.rho * np.maximum(hi - lo, 0.0)


def analytic_sinogram(shapes: Sequence[Shape], angles: np.ndarray, n_det: int,
                      subrays: Sequence[float] = (-0.375, -0.125, 0.125, 0.375)) -> np.ndarray:
    """p[a, d] = mean over sub-rays of the exact line integrals (fp64)."""
    t_d = np.arange(n_det, dtype=np.float64) - (n_det - 1) / 2.0
    th = angles[:, None]
    p = np.zeros((len(angles), n_det), dtype=np.float64)
    for off in subrays:
        t = (t_d + off)[None, :]
        for s in shapes:
            p += (_chord_ellipse(s, th, t) if s.kind == "ellipse" else _chord_rect(s, th, t))
    return p / len(subrays)


def raster(shapes: Sequence[Shape], n: int, supersample: int = 4) -> np.ndarray:
    """Ground-truth image: area average over supersample^2 points per pixel."""
    img = np.zeros((n, n), dtype=np.float64)
    offs = (np.arange(supersample) + 0.5) / supersample - 0.5
    jj = np.arange(n, dtype=np.float64) - (n - 1) / 2.0
    ii = (n - 1) / 2.0 - np.arange(n, dtype=np.float64)
    for oy in offs:
        for ox in offs:
            X = (jj + ox)[None, :]
            Y = (ii - oy)[:, None]
            for s in shapes:
                cp, sp = math.cos(s.phi), math.sin(s.phi)
                u = (X - s.x0) * cp + (Y - s.y0) * sp
                v = -(X - s.x0) * sp + (Y - s.y0) * cp
                if s.kind == "ellipse":
                    inside = (u / s.a) ** 2 + (v / s.b) ** 2 <= 1.0
                else:
                    inside = (np.abs(u) <= s.a) & (np.abs(v) <= s.b)
                img += s.rho * inside
    return img / (supersample * supersample)


def add_noise(p: np.ndarray, kind: str, level: float, rng: np.random.Generator) -> np.ndarray:
    """Gaussian: p + N(0, (level * max p)^2).
    Poisson (reading A16): counts = I0 exp(-p / p_max),
    k ~ Poisson(counts), k <- max(k, 1), p~ = -p_max ln(k / I0); the largest
    expected count is I0 on rays that miss the object."""
    if kind == "gauss":
        return p + rng.normal(0.0, level * float(np.max(p)), size=p.shape)
    if kind == "poisson":
        pmax = float(np.max(p))
        if pmax <= 0.0:
            return p.copy()
        lam = level * np.exp(-p / pmax)
        k = np.maximum(rng.poisson(lam), 1).astype(np.float64)
        return -pmax * np.log(k / level)
    raise ValueError(kind)


def roi_centres(cfg: Config) -> np.ndarray:
    """ROI core centres (row, col) as integer pixel-corner coordinates.
    centre: (N/2, N/2); seeded: uniform integers in [r, N-r]; tiling: r + 2r*I."""
    n, r = cfg.n, cfg.radius
    if cfg.layout == "centre":
        return np.array([[n // 2, n // 2]], dtype=np.int32)
    if cfg.layout == "seeded":
        rng = seeded_rng(cfg.cfg_id, 2)
        return rng.integers(r, n - r + 1, size=(cfg.n_roi, 2)).astype(np.int32)
    if cfg.layout == "sweep":
        rng = seeded_rng(cfg.cfg_id, 2)
        base = rng.integers(r + cfg.margin, n - r - cfg.margin + 1, size=(cfg.n_roi // SWEEP_LAMBDAS, 2))
        return np.repeat(base, SWEEP_LAMBDAS, axis=0).astype(np.int32)
    if cfg.layout == "tiling":
        k = n // (2 * r)
        g = r + 2 * r * np.arange(k)
        rr, cc = np.meshgrid(g, g, indexing="ij")
        out = np.stack([rr.ravel(), cc.ravel()], axis=1).astype(np.int32)
        assert out.shape[0] == cfg.n_roi, (out.shape, cfg.n_roi)
        return out
    raise ValueError(cfg.layout)


@dataclasses.dataclass
class Inputs:
    cfg: Config
    angles: np.ndarray          # fp64 [N_theta]
    shapes: List[Shape]
    sino: np.ndarray            # fp32 [N_theta, N_d]  (noisy, the solver input)
    sino_clean: np.ndarray      # fp64 [N_theta, N_d]
    centres: np.ndarray         # int32 [R, 2]
    sino_trunc: Optional[np.ndarray] = None   # fp32 [N_theta, n_trunc]: the measured central bins


def make_inputs(name_or_cfg, n_angles: Optional[int] = None, n_det: Optional[int] = None,
                n: Optional[int] = None, noise: bool = True) -> Inputs:
    """Full seeded input set for a config (optionally with overridden sizes)."""
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    if n is not None or n_angles is not None or n_det is not None:
        cfg = dataclasses.replace(cfg, n=n or cfg.n, n_angles=n_angles or cfg.n_angles,
                                  n_det=n_det or cfg.n_det)
    ang = angles_for(cfg.n_angles, cfg.span)
    shapes = random_shapes(cfg.n, cfg.n_ellipses, cfg.n_rects, seeded_rng(cfg.cfg_id, 0))
    clean = analytic_sinogram(shapes, ang, cfg.n_det)
    sino = add_noise(clean, cfg.noise, cfg.noise_level, seeded_rng(cfg.cfg_id, 1)) if noise else clean
    trunc = None
    if cfg.n_trunc:
        lo = (cfg.n_det - cfg.n_trunc) // 2
        trunc = np.ascontiguousarray(sino[:, lo:lo + cfg.n_trunc]).astype(np.float32)
    return Inputs(cfg, ang, shapes, sino.astype(np.float32), clean, roi_centres(cfg), trunc)
