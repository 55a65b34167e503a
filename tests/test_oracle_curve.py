"""Pins for the oracle's curve model, residual and row gradient (CPU only).

Model: s = exp(-P_mu) * (f_t * g_Sigma)(m - m_o - z D P_delta), f_t the Gaussian
flat IC A exp(-(m-c)^2/2w^2) (R2), g_Sigma the zero-mean Gaussian of variance P_sigma (R1).
Pins: limits that reduce to the flat curve (north star), numerical quadrature of the
convolution, moment invariants, clamp semantics (R12, R13) and finite differences.
The scattering term has no paper value: it is "parity unpinned" against the paper beyond
these self-consistency pins.
"""
import numpy as np
import pytest
from scipy import integrate

from oracle import ora

ND = 9


def flat_params(rng, nd=ND):
    return (1e4 * (1 + rng.uniform(-0.05, 0.05, nd)), rng.normal(0, 0.05, nd),
            0.15 * (1 + rng.uniform(-0.1, 0.1, nd)))


def flat_curve(A, c, w, m):
    return A * np.exp(-(m - c) ** 2 / (2 * w ** 2))


def test_no_sample_and_attenuation_only_limits():
    rng = np.random.default_rng(0)
    A, c, w = flat_params(rng)
    mask = np.linspace(-0.4, 0.4, 5)
    zero = np.zeros(ND)
    out = ora.curve_row(zero, zero, zero, A, c, w, mask)["s_mod"]
    ref = flat_curve(A[None], c[None], w[None], mask[:, None])          # maps 0 -> s = f
    np.testing.assert_allclose(out, ref, rtol=2e-16 * 8)
    # sigma = 0 and Delta = 0 (P_delta constant along t) -> s = exp(-P_mu) f  (north star)
    p_mu = rng.uniform(0, 0.5, ND)
    out = ora.curve_row(p_mu, np.full(ND, 0.37), zero, A, c, w, mask)["s_mod"]
    np.testing.assert_allclose(out, np.exp(-p_mu)[None] * ref, rtol=2e-16 * 16)


def test_broadening_is_gaussian_convolution():
    """s(m) = T int f(m - m_o - Delta - tau) g_Sigma(tau) dtau, by adaptive quadrature."""
    rng = np.random.default_rng(1)
    A, c, w = flat_params(rng)
    p_mu = rng.uniform(0, 0.3, ND)
    slope = 0.021
    p_delta = slope * np.arange(ND)                     # D P_delta = slope exactly (ramp)
    p_sigma = (rng.uniform(0.02, 0.2, ND) * 0.15) ** 2  # Sigma in [0.02, 0.2] widths
    z, drift = 1.7, -0.013
    mask = np.array([-0.33, -0.1, 0.0, 0.21, 0.4])
    out = ora.curve_row(p_mu, p_delta, p_sigma, A, c, w, mask, drift=drift, z=z)["s_mod"]
    for k in range(ND):
        sig = np.sqrt(p_sigma[k])
        for j, m in enumerate(mask):
            arg = m - drift - z * slope
            f = lambda tau: (flat_curve(A[k], c[k], w[k], arg - tau) *
                             np.exp(-tau ** 2 / (2 * sig ** 2)) / np.sqrt(2 * np.pi * sig ** 2))
            val, _ = integrate.quad(f, -12 * sig, 12 * sig, epsabs=0, epsrel=1e-13, limit=200)
            ref = np.exp(-p_mu[k]) * val
            assert abs(out[j, k] - ref) <= 1e-10 * abs(ref) + 1e-12


def test_moment_invariants():
    """On a fine m grid: int s dm = T A w sqrt(2 pi) (independent of Delta, Sigma);
    centroid = c + m_o + Delta (positive Delta moves the peak to larger m, R10); variance = W^2."""
    rng = np.random.default_rng(2)
    A, c, w = flat_params(rng, 5)
    p_mu = rng.uniform(0, 0.3, 5)
    p_delta = 0.03 * np.arange(5) ** 2              # D P_delta = [0.03, 0.06, 0.12, 0.18, 0.21]
    p_sigma = (np.array([0.0, 0.05, 0.1, 0.15, 0.2]) * 0.15) ** 2
    z, drift = 1.0, 0.02
    dm = 1e-3
    grid = np.arange(-4.0, 4.0, dm)
    s = ora.curve_row(p_mu, p_delta, p_sigma, A, c, w, grid, drift=drift, z=z)["s_mod"]
    Dp = np.array([0.03, 0.06, 0.12, 0.18, 0.21])   # hand-computed D of 0.03 k^2 (one-sided ends)
    area = s.sum(axis=0) * dm
    np.testing.assert_allclose(area, np.exp(-p_mu) * A * w * np.sqrt(2 * np.pi), rtol=1e-8)
    cen = (s * grid[:, None]).sum(axis=0) * dm / area
    np.testing.assert_allclose(cen, c + drift + z * Dp, rtol=0, atol=1e-8)
    var = (s * (grid[:, None] - cen) ** 2).sum(axis=0) * dm / area
    np.testing.assert_allclose(var, w ** 2 + p_sigma, rtol=1e-8)


def test_clamps_and_counters():
    """R12: P_mu clamped to [-50, 50] with zero mu-gradient there; R13: W^2 >= w^2/100 with zero
    sigma-gradient there; both counted."""
    A, c, w = np.full(4, 1e4), np.zeros(4), np.full(4, 0.15)
    p_mu = np.array([0.1, 60.0, -70.0, 0.2])
    p_sigma = np.array([0.0, 0.0, 0.0, -0.15 ** 2])
    mask = np.array([-0.2, 0.0, 0.2])
    s_exp = np.ones((3, 4))
    out = ora.curve_row(p_mu, np.zeros(4), p_sigma, A, c, w, mask, s_exp=s_exp)
    assert list(out["counters"]) == [2, 1]
    np.testing.assert_allclose(out["s_mod"][:, 1], np.exp(-50.0) * flat_curve(1e4, 0, 0.15, mask),
                               rtol=1e-14)
    W2 = 0.15 ** 2 / 100
    np.testing.assert_allclose(out["s_mod"][:, 3],
                               np.exp(-0.2) * 1e4 * 0.15 / np.sqrt(W2) * np.exp(-mask ** 2 / (2 * W2)),
                               rtol=1e-14)
    assert out["g_mu"][1] == 0 and out["g_mu"][2] == 0 and out["g_mu"][0] != 0
    assert out["g_sigma"][3] == 0 and out["g_sigma"][0] != 0


@pytest.mark.parametrize("z,du", [(1.0, 1.0), (2.3, 0.7)])
def test_row_gradient_finite_differences(z, du):
    """dS/dP from curve_row (incl. z D^T) against central differences of its own cost."""
    rng = np.random.default_rng(3)
    nd = 11
    A, c, w = flat_params(rng, nd)
    p = [rng.uniform(0, 0.3, nd), rng.uniform(0, 0.05, nd), (rng.uniform(0, 0.2, nd) * 0.15) ** 2]
    mask = np.linspace(-0.4, 0.4, 6)
    s_exp = rng.poisson(flat_curve(A[None], c[None], w[None], mask[:, None]) * 0.8).astype(float)
    base = ora.curve_row(*p, A, c, w, mask, drift=0.01, z=z, du=du, s_exp=s_exp)
    grads = [base["g_mu"], base["g_delta"], base["g_sigma"]]
    for q in range(3):
        h = 1e-6 * max(np.abs(p[q]).max(), 1e-3)
        fd = np.zeros(nd)
        for k in range(nd):
            pp = [x.copy() for x in p]
            pm = [x.copy() for x in p]
            pp[q][k] += h
            pm[q][k] -= h
            cp = ora.curve_row(*pp, A, c, w, mask, drift=0.01, z=z, du=du, s_exp=s_exp)["cost"]
            cm = ora.curve_row(*pm, A, c, w, mask, drift=0.01, z=z, du=du, s_exp=s_exp)["cost"]
            fd[k] = (cp - cm) / (2 * h)
        assert np.linalg.norm(fd - grads[q]) / np.linalg.norm(grads[q]) < 1e-6, q
