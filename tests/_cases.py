"""Oracle-built test cases (tests only).  Inputs come from paper_2202_08627_b200.synth (draws,
no method arithmetic) and the fp64 oracle (scaling per R16 and the noise-free model per R20);
nothing here ever comes from the CUDA path."""
import functools

import numpy as np

from oracle import ora
from paper_2202_08627_b200 import synth


def oracle_case(cfg: synth.Config, with_data: bool = True, noise: bool = True) -> synth.Case:
    ang = cfg.angles

    def max_shift(delta):
        P = ora.project(delta, ang, cfg.n_det, cfg.pixel, cfg.det_pitch)
        return float(max(np.abs(cfg.z * ora.diff_t(row, cfg.det_pitch)).max() for row in P))

    def max_proj(img):
        return float(ora.project(img, ang, cfg.n_det, cfg.pixel, cfg.det_pitch).max())

    def model(case):
        smod, _ = ora.forward(ang, case.mu, case.delta, case.sigma, case.flat, case.mask, case.drift,
                              dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z)
        return smod

    return synth.make_case(cfg, max_shift, max_proj, model if with_data else None, noise=noise)


@functools.lru_cache(maxsize=None)
def cached_case(name: str) -> synth.Case:
    if name in synth.CONFIGS:
        return oracle_case(synth.CONFIGS[name])
    if name == "R1":
        return oracle_case(synth.small_config())
    if name == "R2":   # 180-degree span, even sizes, no drift, M=1 (the paper's single-offset case)
        return oracle_case(synth.small_config("R2", S=1, N=40, n_angles=24, span_deg=180.0, n_det=58,
                                              M=1, K=4, drift_sd=0.0, w_jit=0.0, texture=0.0, seed=91))
    if name == "R3":   # 360-degree scan with an even angle count: mirror pairs (theta, theta + pi)
        return oracle_case(synth.small_config("R3", S=2, N=48, n_angles=40, span_deg=360.0, n_det=70,
                                              M=3, K=5, drift_sd=0.002, w_jit=0.1, texture=0.05, seed=95))
    raise KeyError(name)


def oracle_cost_grad(case: synth.Case, maps, lam=0.0, slices=None):
    cfg = case.cfg
    return ora.cost_grad(cfg.angles, *maps, case.flat, case.mask, case.drift, case.s_exp, lam,
                         dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z, slices=slices)


def oracle_h_case(cfg: synth.Config, gamma: float = synth.H_GAMMA, noise: bool = True) -> synth.HCase:
    """Single-map model case (NEXT-3): z from the oracle projector, s_exp = Poisson(oracle model)."""
    ang = cfg.angles

    def max_shift(img):
        P = ora.project(img, ang, cfg.n_det, cfg.pixel, cfg.det_pitch)
        return float(max(np.abs(ora.diff_t(row, cfg.det_pitch)).max() for row in P))

    def model(case):
        c = case.cfg
        return ora.cost_grad_h(ang, case.h, case.gamma, case.flat, case.mask, case.drift,
                               dx=c.pixel, du=c.det_pitch, z=c.z)

    return synth.make_h_case(cfg, gamma, max_shift, model, noise=noise)


@functools.lru_cache(maxsize=None)
def cached_h_case(name: str) -> synth.HCase:
    if name in synth.H_CONFIGS:
        return oracle_h_case(synth.H_CONFIGS[name])
    if name == "RH":   # ragged: odd sizes, detector narrower than the map diagonal, drift, M = 2
        return oracle_h_case(synth.small_config("RH", S=2, N=41, n_angles=29, span_deg=360.0, n_det=47,
                                                M=2, K=4, drift_sd=0.003, w_jit=0.1, texture=0.0,
                                                seed=93))
    raise KeyError(name)


def oracle_cost_grad_h(case: synth.HCase, h, lam=0.0):
    c = case.cfg
    return ora.cost_grad_h(c.angles, h, case.gamma, case.flat, case.mask, case.drift, case.s_exp, lam,
                           dx=c.pixel, du=c.det_pitch, z=c.z)


@functools.lru_cache(maxsize=None)
def cached_hs_case(name: str, n_knots: int = 33):
    """Single-map case with the sampled flat IC (NEXT-4): flat_samples from 20 averaged Poisson
    scans of 33 steps of the case's Gaussian IC; s_exp = Poisson(oracle sampled-IC model)."""
    base = cached_h_case(name)
    c = base.cfg
    fs = synth.sampled_flat(base.flat, n_knots, repeats=20, seed=c.seed + 31)
    smod = ora.cost_grad_hs(c.angles, base.h, base.gamma, fs, base.mask, base.drift,
                            dx=c.pixel, du=c.det_pitch, z=c.z)
    rng = np.random.default_rng(c.seed + 32)
    s_exp = rng.poisson(np.maximum(smod, 0.0)).astype(np.float32)
    return base, fs, s_exp


def oracle_objective(case: synth.Case, lam: float = 0.0):
    """fg(x) over x = [3, S, N, N] (CPU fp64 tensors) with the fp64 oracle's cost and gradient:
    the same objective the product path evaluates on the GPU (lbfgs.ei_objective)."""
    import torch
    cfg = case.cfg

    def fg(x):
        m = x.numpy()
        c, gm, gd, gs, _ = ora.cost_grad(cfg.angles, m[0], m[1], m[2], case.flat, case.mask, case.drift,
                                         case.s_exp, lam, dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z)
        return torch.from_numpy(c), torch.from_numpy(np.stack([gm, gd, gs]))
    return fg


def oracle_objective_drift(case: synth.Case, lam: float = 0.0, slices=None):
    """fg over the blocks [mu, delta, sigma, m_o] of a stack treated as ONE problem (joint drift
    estimation, R25): mu/delta/sigma [1, S, N, N], m_o [1, N_theta]; cost = sum over slices,
    dS/dm_o = sum over slices of the oracle's per-slice drift gradient.  `slices`: evaluate only
    these slices of the case (one rank's shard)."""
    import torch
    cfg = case.cfg
    sl = list(range(cfg.S)) if slices is None else list(slices)

    def fg(x):
        mu, de, sg, mo = (b.numpy() for b in x)
        full = [np.zeros((cfg.S,) + mu.shape[2:], np.float64) for _ in range(3)]
        for q, b in enumerate((mu, de, sg)):
            full[q][sl] = b[0]
        c, gm, gd, gs, _, gdr = ora.cost_grad(cfg.angles, *full, case.flat, case.mask,
                                              mo[0].astype(np.float32), case.s_exp, lam, dx=cfg.pixel,
                                              du=cfg.det_pitch, z=cfg.z, slices=sl, want_drift=True)
        return (torch.tensor([c.sum()], dtype=torch.float64),
                [torch.from_numpy(gm)[None], torch.from_numpy(gd)[None], torch.from_numpy(gs)[None],
                 torch.from_numpy(gdr.sum(0))[None]])
    return fg


def rms_of_range(x, truth, border: int = 2) -> float:
    """SPEC.md:562 (acceptance 9): RMS error excluding a `border`-pixel frame, as a fraction of the
    phantom's dynamic range."""
    d = (np.asarray(x, np.float64) - truth)[..., border:-border, border:-border]
    return float(np.sqrt((d ** 2).mean()) / (truth.max() - truth.min()))


def drift_rms(est, truth) -> float:
    """drift error RMS up to a global constant, relative to the drift's own RMS about
    its mean."""
    d = np.asarray(est, np.float64) - truth
    d = d - d.mean()
    t = truth - truth.mean()
    return float(np.sqrt((d ** 2).mean()) / np.sqrt((t ** 2).mean()))
