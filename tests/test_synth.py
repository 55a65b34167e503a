"""Generator recipe checks (readings R15-R21) — CPU only."""
import numpy as np

from oracle import ora
from paper_2202_08627_b200 import synth
import _cases


def test_c1_recipe_targets():
    case = _cases.cached_case("C1")
    cfg = case.cfg
    assert case.mu.dtype == np.float32 and case.s_exp.dtype == np.float32
    assert abs(case.mu.max() - 0.02) < 1e-8                                  # R17
    P = ora.project(case.delta[0].astype(np.float64), cfg.angles, cfg.n_det)
    shift = max(np.abs(ora.diff_t(r)).max() for r in P)
    assert abs(shift - 0.3 * cfg.w0) < 1e-6                                   # R16
    Ps = ora.project(case.sigma[0].astype(np.float64), cfg.angles, cfg.n_det)
    assert abs(np.sqrt(Ps.max()) - 0.2 * cfg.w0) < 1e-6                       # R16 / R1-B
    np.testing.assert_allclose(case.mask, [-0.4, -0.2, 0.0, 0.2, 0.4], atol=1e-7)   # R3
    assert np.all(case.s_exp >= 0) and np.all(case.s_exp == np.round(case.s_exp))  # Poisson
    A, c, w = case.flat[0]
    assert np.all(np.abs(A / 1e4 - 1) <= 0.05 + 1e-6) and np.allclose(w, 0.15)    # R15


def test_deterministic_and_drift():
    cfg = synth.small_config()
    a, _ = synth.draw_slice(cfg, 1)
    b, _ = synth.draw_slice(cfg, 1)
    assert np.array_equal(a.mu, b.mu) and np.array_equal(a.flat, b.flat)
    d = synth.draw_drift(cfg)
    assert d[0] == 0 and d.shape == (cfg.n_angles,)
    assert synth.draw_drift(synth.CONFIGS["C1"]) is None
    c4 = synth.CONFIGS["C4"]
    assert c4.S == 64 and c4.N == 512 and c4.n_angles == 720 and c4.n_det == 768 and c4.M == 7


def test_paper_workload_config():
    """P1 follows the paper's scan: 220 x 220, 400 angles over 360 deg, one mask
    position at 9 um from the IC maximum with a 38 um period."""
    cfg = synth.H_CONFIGS["P1"]
    assert (cfg.N, cfg.n_angles, cfg.n_det, cfg.M) == (220, 400, 220, 1)
    assert np.isclose(np.rad2deg(cfg.angles[-1] + cfg.angles[1]), 360.0)
    assert np.isclose(cfg.mask[0], 9.0 / 38.0)
    assert synth.H_GAMMA == 5.0 and synth.H_LAMBDA == 1e-2
