"""Pins for the oracle's sampled flat IC (NEXT-4; "scanned over one period with 33
steps", read between the samples by a periodic Catmull-Rom cubic, reading R23 from SPEC.md:147-159)
and for the single-map model built on it — CPU only.

* knot reproduction and periodicity
* quadratic precision: Catmull-Rom reproduces any quadratic between interior knots exactly
  (a textbook property of its finite-difference tangents) — pins every cubic coefficient
* analytic cosine within 1e-3 (33 knots) and its derivative; f' against central
  differences of f
* the model's gradient against central differences of its cost, and convergence to the
  parametric Gaussian model (ora.cost_grad_h) as the knots get denser
"""
import numpy as np
import pytest

from oracle import ora
from paper_2202_08627_b200 import synth

from test_oracle_gradient import tiny_problem


def table(fun, K, nd=3):
    m = np.arange(K) / K
    return np.stack([fun(m) * (1 + 0.1 * t) for t in range(nd)], axis=1).astype(np.float32)


def test_knots_and_periodicity():
    rng = np.random.default_rng(0)
    fs = rng.uniform(0, 1e4, (32, 4)).astype(np.float32)
    for q in range(32):
        for t in range(4):
            f, _ = ora.ic_eval(fs, t, q / 32.0)
            assert f == pytest.approx(float(fs[q, t]), rel=1e-13, abs=1e-9)
    for m in rng.uniform(0, 1, 20):
        a = ora.ic_eval(fs, 2, m)
        for k in (-2, -1, 1, 3):
            b = ora.ic_eval(fs, 2, m + k)
            assert b[0] == pytest.approx(a[0], rel=1e-11) and b[1] == pytest.approx(a[1], rel=1e-9)


def test_quadratic_precision():
    K = 40
    q = lambda m: 3.0 - 2.0 * m + 7.5 * m * m                    # sampled on the knots
    fs = np.asarray(q(np.arange(K) / K), np.float64)[:, None].astype(np.float32)
    for m in np.linspace(2.0 / K, (K - 3.0) / K, 57):            # interior: no periodic wrap
        f, fp = ora.ic_eval(fs, 0, m)
        # fp32 knots: compare with the quadratic through the rounded samples' scale
        assert f == pytest.approx(q(m), rel=2e-6)
        assert fp == pytest.approx(-2.0 + 15.0 * m, rel=2e-4, abs=2e-4)


def test_cosine_and_derivative():
    K = 33
    fs = table(lambda m: 1.0 + 0.5 * np.cos(2 * np.pi * m), K)
    for m in np.random.default_rng(1).uniform(0, 1, 50):
        f, fp = ora.ic_eval(fs, 0, m)
        assert abs(f - (1 + 0.5 * np.cos(2 * np.pi * m))) <= 1e-3 * 1.5
        assert abs(fp - (-np.pi * np.sin(2 * np.pi * m))) <= 1e-2 * np.pi
        e = 1e-3 / K
        fd = (ora.ic_eval(fs, 0, m + e)[0] - ora.ic_eval(fs, 0, m - e)[0]) / (2 * e)
        assert fd == pytest.approx(fp, rel=1e-6, abs=1e-6)


def _cost64_hs(ang, h64, gamma, fs, mask, drift, s_exp, z):
    """fp64 cost of the sampled-IC model via project + ic_eval (the same definitions, a different
    route through the code than ora.cost_grad_hs's fused loop)."""
    na, m, nd = s_exp.shape[1:]
    P = ora.project(h64, ang, nd)
    S = 0.0
    for a in range(na):
        dP = ora.diff_t(P[a])
        for k in range(nd):
            T = np.exp(-P[a][k])
            for j in range(m):
                f, _ = ora.ic_eval(fs[0], k, float(mask[j]) - float(drift[a]) - z * gamma * dP[k])
                S += (T * f - float(s_exp[0, a, j, k])) ** 2
    return S


def test_hs_gradient_matches_finite_differences():
    ang, maps, flat, mask, drift, s_exp = tiny_problem(11, n=5, na=4, nd=8, m=2)
    fs = synth.sampled_flat(flat, 33, seed=3)
    h = maps[0]
    gamma, z = 5.0, 1.0
    cost, grad, st = ora.cost_grad_hs(ang, h, gamma, fs, mask, drift, s_exp, 0.0, z=z)
    h64 = h[0].astype(np.float64)
    assert _cost64_hs(ang, h64, gamma, fs, mask, drift, s_exp, z) == pytest.approx(cost[0], rel=1e-12)
    step = 1e-4 * np.abs(h64).max()
    fd = np.zeros_like(h64)
    for idx in np.ndindex(*h64.shape):
        hp, hm = h64.copy(), h64.copy()
        hp[idx] += step
        hm[idx] -= step
        fd[idx] = (_cost64_hs(ang, hp, gamma, fs, mask, drift, s_exp, z) -
                   _cost64_hs(ang, hm, gamma, fs, mask, drift, s_exp, z)) / (2 * step)
    assert np.linalg.norm(fd - grad[0]) / np.linalg.norm(grad[0]) < 1e-6


def test_sampled_model_converges_to_parametric_model():
    """Noise-free samples of a narrow Gaussian IC: the sampled-IC model approaches the parametric
    one as the knots get denser (third-order Catmull-Rom: ~8x per doubling).  The mask span and
    gamma keep every IC argument within 0.3 periods of the centre, where the periodic images of
    the sampled curve are < 1e-10 of its peak."""
    ang, maps, flat, mask, drift, s_exp = tiny_problem(12, n=8, na=6, nd=12, m=3)
    flat = flat.copy()
    flat[:, 2] = 0.1
    mask = np.linspace(-0.15, 0.15, 3).astype(np.float32)
    h = maps[0]
    ref = ora.cost_grad_h(ang, h, 1.0, flat, mask, drift)
    errs = []
    for K in (33, 66, 132):
        fs = synth.sampled_flat(flat, K, noise=False)
        sm = ora.cost_grad_hs(ang, h, 1.0, fs, mask, drift)
        errs.append(np.linalg.norm(sm - ref) / np.linalg.norm(ref))
    assert errs[0] < 2e-3 and errs[1] < errs[0] / 4 and errs[2] < errs[1] / 4, errs
