"""Seeded synthetic inputs shaped like the paper's scans (BASELINE.json configs C1-C5).

This module holds NO arithmetic of the method (no projector, no curve model, no cost):
it draws phantoms, flat-IC parameters, mask positions, drift and Poisson noise.  The two
steps of the recipe that need the forward model — scaling delta/sigma to a target
refraction shift / broadening (reading R16) and the noise-free curves that Poisson noise
is drawn around (R20) — take the model as an argument: tests pass the fp64 oracle, bench.py
passes the product path.  It is the only code shared by the oracle side and the CUDA side.

Recipe (frozen from SURVEY.md §8(c) R15-R21 and §8(d)):
  * angles theta_a = a * span / N_theta (uniform, span 180 or 360 deg)
  * mask positions m_j = (j - (M-1)/2) / M, period units (R3)
  * K random ellipses (R18), 4x4 supersampled raster; mu, delta, sigma share shapes
    with independent per-ellipse values U[0,1)
  * mu scaled so max mu = 0.02 * 64 / N (R17); delta so max |z D R[delta]| = 0.3 w0 and
    sigma so max R[sigma] = (0.2 w0)^2 (R16, R1-B)
  * flat IC per detector pixel: A = A0 (1 + U[-5%, 5%]), c ~ N(0, 0.05), w = w0 (1 + U[-wj, wj])
  * drift (C4): random walk m_o(0) = 0, steps N(0, 0.002) (R14)
  * C3 texture on delta: U[-a, a], a = 5% of max delta, inside the ellipse union (R19)
  * s_exp = Poisson(s_mod(truth)) stored as fp32 (R20)
Draw order: ellipses -> map values -> flat params -> drift -> texture -> Poisson.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Optional

import numpy as np


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    S: int            # slices
    N: int            # grid N x N
    n_angles: int
    span_deg: float
    n_det: int
    M: int            # mask positions
    K: int            # ellipses
    A0: float         # flat amplitude (counts)
    w0: float         # nominal flat width (periods)
    w_jit: float      # relative width jitter (uniform)
    texture: float    # delta texture amplitude (fraction of max)
    drift_sd: float   # per-angle drift random-walk step (periods)
    seed: int
    pixel: float = 1.0
    det_pitch: float = 1.0
    z: float = 1.0
    mask_offset: float = 0.0   # added to every mask position (P1: the paper's slope position)

    @property
    def angles(self) -> np.ndarray:
        return np.arange(self.n_angles, dtype=np.float64) * np.deg2rad(self.span_deg) / self.n_angles

    @property
    def mask(self) -> np.ndarray:
        return ((np.arange(self.M) - (self.M - 1) / 2.0) / self.M + self.mask_offset).astype(np.float32)


# BASELINE.json configs[0..4]
CONFIGS = {
    "C1": Config("C1", 1, 64, 90, 180.0, 96, 5, 8, 1e4, 0.15, 0.0, 0.0, 0.0, 1000),
    "C2": Config("C2", 1, 256, 360, 180.0, 384, 7, 8, 1e4, 0.15, 0.0, 0.0, 0.0, 2000),
    "C3": Config("C3", 1, 1024, 1440, 360.0, 1536, 9, 32, 5e3, 0.15, 0.10, 0.05, 0.0, 3000),
    "C4": Config("C4", 64, 512, 720, 180.0, 768, 7, 8, 1e4, 0.15, 0.0, 0.0, 0.002, 4000),
    "C5": Config("C5", 1, 2048, 240, 180.0, 3072, 5, 64, 2e3, 0.12, 0.0, 0.0, 0.0, 5000),
}

# The paper's own scan geometry for its single-map model (NEXT-3): a 220 x 220
# slice (N_t = 220 detector pixels), 400 projections over 360 deg, one mask position on the slope
# of the IC, 9 um from its maximum with a 38 um sample-mask period (m = 9/38 period), gamma = 5,
# lambda = 1e-2.  The plastic-granule phantom is a seeded sum of 12 ellipses (the real scan is
# not in the container).
H_CONFIGS = {
    "P1": Config("P1", 1, 220, 400, 360.0, 220, 1, 12, 1e4, 0.15, 0.0, 0.0, 0.0, 6000,
                 mask_offset=9.0 / 38.0),
}
H_GAMMA = 5.0
H_LAMBDA = 1e-2


def small_config(name="R1", S=2, N=67, n_angles=37, span_deg=360.0, n_det=101, M=3, K=5,
                 drift_sd=0.002, w_jit=0.1, texture=0.05, seed=77) -> Config:
    """Ragged test geometry (odd sizes, partial tiles, drift, texture) for parity tests."""
    return Config(name, S, N, n_angles, span_deg, n_det, M, K, 1e4, 0.15, w_jit, texture, drift_sd, seed)


def with_slices(cfg: Config, S: int) -> Config:
    return dataclasses.replace(cfg, S=S)


# --------------------------------------------------------------------------------------
# phantom
# --------------------------------------------------------------------------------------
def draw_ellipses(rng: np.random.Generator, N: int, K: int) -> np.ndarray:
    """R18: rows (a, b, phi, x0, y0) in pixel units relative to the grid centre."""
    out = np.zeros((K, 5))
    for e in range(K):
        a, b = rng.uniform(0.05, 0.3, size=2) * N / 2
        phi = rng.uniform(0, np.pi)
        rad = rng.uniform(0, 0.9 * N / 2 - max(a, b))
        ang = rng.uniform(0, 2 * np.pi)
        out[e] = (a, b, phi, rad * np.cos(ang), rad * np.sin(ang))
    return out


def raster_ellipse(N: int, ell, sub: int = 4) -> tuple:
    """Coverage fraction of one ellipse on the N x N grid (sub x sub supersampling), returned
    as (i0, j0, block) restricted to the ellipse's bounding box."""
    a, b, phi, x0, y0 = ell
    r = max(a, b) + 1.0
    ctr = (N - 1) / 2.0
    i0 = max(int(np.floor(y0 + ctr - r)), 0)
    i1 = min(int(np.ceil(y0 + ctr + r)) + 1, N)
    j0 = max(int(np.floor(x0 + ctr - r)), 0)
    j1 = min(int(np.ceil(x0 + ctr + r)) + 1, N)
    if i1 <= i0 or j1 <= j0:
        return i0, j0, np.zeros((0, 0))
    ys = (np.arange(i0, i1) - ctr)[:, None]
    xs = (np.arange(j0, j1) - ctr)[None, :]
    cphi, sphi = np.cos(phi), np.sin(phi)
    cover = np.zeros((i1 - i0, j1 - j0))
    offs = (np.arange(sub) + 0.5) / sub - 0.5
    for oy in offs:
        for ox in offs:
            dx, dy = xs + ox - x0, ys + oy - y0
            xr = dx * cphi + dy * sphi
            yr = -dx * sphi + dy * cphi
            cover += ((xr / a) ** 2 + (yr / b) ** 2 <= 1.0)
    return i0, j0, cover / (sub * sub)


def raster(N: int, ellipses: np.ndarray, values: np.ndarray) -> np.ndarray:
    img = np.zeros((N, N))
    for ell, v in zip(ellipses, values):
        i0, j0, blk = raster_ellipse(N, ell)
        img[i0:i0 + blk.shape[0], j0:j0 + blk.shape[1]] += v * blk
    return img


@dataclasses.dataclass
class Slice:
    mu: np.ndarray
    delta: np.ndarray
    sigma: np.ndarray
    flat: np.ndarray      # [3][Nd]: A, c, w


def draw_slice(cfg: Config, s: int) -> tuple:
    """Unscaled maps + flat parameters for slice s, plus the rng (for later draws)."""
    rng = np.random.default_rng(cfg.seed + s)
    ell = draw_ellipses(rng, cfg.N, cfg.K)
    vals = rng.uniform(0.0, 1.0, size=(3, cfg.K))
    mu, delta, sigma = (raster(cfg.N, ell, vals[q]) for q in range(3))
    A = cfg.A0 * (1.0 + rng.uniform(-0.05, 0.05, cfg.n_det))
    c = rng.normal(0.0, 0.05, cfg.n_det)
    w = cfg.w0 * (1.0 + (rng.uniform(-cfg.w_jit, cfg.w_jit, cfg.n_det) if cfg.w_jit > 0 else 0.0))
    flat = np.stack([A, c, np.broadcast_to(w, (cfg.n_det,))]).astype(np.float32)
    if cfg.texture > 0:
        inside = np.zeros((cfg.N, cfg.N), bool)
        for e in ell:
            i0, j0, blk = raster_ellipse(cfg.N, e)
            inside[i0:i0 + blk.shape[0], j0:j0 + blk.shape[1]] |= blk > 0
        amp = cfg.texture * delta.max()
        delta = delta + np.where(inside, rng.uniform(-amp, amp, (cfg.N, cfg.N)), 0.0)
    return Slice(mu, delta, sigma, flat), rng


def draw_drift(cfg: Config) -> Optional[np.ndarray]:
    if cfg.drift_sd <= 0:
        return None
    rng = np.random.default_rng(cfg.seed + 999)
    steps = rng.normal(0.0, cfg.drift_sd, cfg.n_angles)
    steps[0] = 0.0
    return np.cumsum(steps).astype(np.float32)


@dataclasses.dataclass
class Case:
    cfg: Config
    mu: np.ndarray        # [S][N][N] fp32 (truth)
    delta: np.ndarray
    sigma: np.ndarray
    flat: np.ndarray      # [S][3][Nd] fp32
    mask: np.ndarray      # [M] fp32
    drift: Optional[np.ndarray]   # [Na] fp32 or None
    s_exp: Optional[np.ndarray] = None   # [S][Na][M][Nd] fp32

    @property
    def angles(self):
        return self.cfg.angles

    def maps(self):
        return self.mu, self.delta, self.sigma


def make_case(cfg: Config,
              max_shift: Callable[[np.ndarray], float],
              max_proj: Callable[[np.ndarray], float],
              model: Optional[Callable[["Case"], np.ndarray]] = None, noise: bool = True) -> Case:
    """Build the truth maps (scaled per R16/R17) and, if ``model`` is given, s_exp = Poisson(model).

    max_shift(delta_2d) must return max |z D R[delta]|; max_proj(img_2d) max R[img];
    model(case) must return s_mod [S][Na][M][Nd] for the case's truth maps.  noise=False stores the
    noise-free curves (exact-fit experiments)."""
    S, N = cfg.S, cfg.N
    mu = np.zeros((S, N, N), np.float32)
    delta = np.zeros_like(mu)
    sigma = np.zeros_like(mu)
    flat = np.zeros((S, 3, cfg.n_det), np.float32)
    rngs = []
    for s in range(S):
        sl, rng = draw_slice(cfg, s)
        rngs.append(rng)
        m = sl.mu * ((0.02 * 64 / N) / max(sl.mu.max(), 1e-30))
        d = sl.delta * (0.3 * cfg.w0 / max(max_shift(sl.delta), 1e-30))
        g = sl.sigma * ((0.2 * cfg.w0) ** 2 / max(max_proj(sl.sigma), 1e-30))
        mu[s], delta[s], sigma[s], flat[s] = m, d, g, sl.flat
    case = Case(cfg, mu, delta, sigma, flat, cfg.mask, draw_drift(cfg))
    if model is not None:
        smod = np.asarray(model(case), dtype=np.float64)
        s_exp = np.empty(smod.shape, np.float32)
        for s in range(S):
            s_exp[s] = (rngs[s].poisson(np.maximum(smod[s], 0.0)) if noise else smod[s]).astype(np.float32)
        case.s_exp = s_exp
    return case


def perturbed(maps, seed: int, rel: float = 0.1):
    """R21: x_pert = x_true * (1 + rel * U[-1, 1]) (seeded)."""
    rng = np.random.default_rng(seed)
    return tuple((m * (1.0 + rel * rng.uniform(-1, 1, m.shape))).astype(np.float32) for m in maps)


def uniform(shape, seed: int) -> np.ndarray:
    """Nonnegative U[0,1) vectors for dot tests."""
    return np.random.default_rng(seed).uniform(0.0, 1.0, shape).astype(np.float32)


@dataclasses.dataclass
class HCase:
    """Inputs of the single-map model (NEXT-3): truth h, flat, mask, drift, gamma, s_exp; cfg.z is
    set so that the largest refraction shift z gamma |D R[h]| is 0.3 nominal IC widths (R16's
    recipe applied to delta = gamma h)."""
    cfg: Config
    h: np.ndarray                 # [S][N][N] fp32 (truth)
    gamma: float
    flat: np.ndarray              # [S][3][Nd]
    mask: np.ndarray              # [M]
    drift: Optional[np.ndarray]
    s_exp: Optional[np.ndarray] = None


def make_h_case(cfg: Config, gamma: float,
                max_shift: Callable[[np.ndarray], float],
                model: Optional[Callable[["HCase"], np.ndarray]] = None, noise: bool = True) -> HCase:
    """max_shift(img_2d) must return max |D R[img]| (unit z); model(case) s_mod [S][Na][M][Nd]."""
    S, N = cfg.S, cfg.N
    h = np.zeros((S, N, N), np.float32)
    flat = np.zeros((S, 3, cfg.n_det), np.float32)
    rngs = []
    for s in range(S):
        sl, rng = draw_slice(cfg, s)
        rngs.append(rng)
        h[s] = sl.mu * ((0.02 * 64 / N) / max(sl.mu.max(), 1e-30))      # R17 scale on mu = h
        flat[s] = sl.flat
    shift = max(max_shift(h[s]) for s in range(S))
    z = 0.3 * cfg.w0 / max(gamma * shift, 1e-30)
    case = HCase(dataclasses.replace(cfg, z=float(z)), h, float(gamma), flat, cfg.mask, draw_drift(cfg))
    if model is not None:
        smod = np.asarray(model(case), dtype=np.float64)
        s_exp = np.empty(smod.shape, np.float32)
        for s in range(S):
            s_exp[s] = (rngs[s].poisson(np.maximum(smod[s], 0.0)) if noise else smod[s]).astype(np.float32)
        case.s_exp = s_exp
    return case


def sampled_flat(flat: np.ndarray, n_knots: int = 33, repeats: int = 20, seed: int = 0,
                 noise: bool = True) -> np.ndarray:
    """A measured flat IC (NEXT-4): the paper scans the sample mask over one period in 33 steps
    and repeats the scan 20 times.  Synthesised here per detector pixel from the
    Gaussian flat parameters flat [S][3][Nd] = (A, c, w) as the periodic curve of one mask period,
    A sum_k exp(-(m_q - c - k)^2 / (2 w^2)) at m_q = q / n_knots, Poisson-sampled `repeats` times
    and averaged.  Returns [S][n_knots][Nd] fp32."""
    rng = np.random.default_rng(seed)
    A, c, w = (flat[:, q, None, :].astype(np.float64) for q in range(3))
    m = (np.arange(n_knots) / n_knots)[None, :, None]
    f = sum(A * np.exp(-(m - c - k) ** 2 / (2 * w * w)) for k in (-2, -1, 0, 1, 2))
    if noise:
        f = sum(rng.poisson(f) for _ in range(repeats)) / repeats
    return f.astype(np.float32)
