"""Pins for the oracle's single-map model (NEXT-3): eq. 4 with m_r = 0
under the homogeneity assumption mu = gamma^-1 delta = h, cost eq. 5 — CPU only.

* the gradient against central finite differences of an fp64 cost evaluated through a different
  route (the three-map row function with P_delta = gamma P_h, P_sigma = 0), on N = 6 grids
* the model is the three-map model at (mu, delta, sigma) = (h, gamma h, 0): equal cost, and
  grad_h = grad_mu + gamma grad_delta (chain rule)
* gamma = 0 removes the refraction: s_mod = T f exactly (eq. 2 with delta = 0)
* exact fit: s_exp = s_mod(h) -> S and grad vanish up to the fp32 rounding of s_exp
"""
import numpy as np
import pytest

from oracle import ora

from test_oracle_gradient import tiny_problem


def _cost64(ang, h64, gamma, flat, mask, drift, s_exp, lam, z):
    na, m, nd = s_exp.shape[1:]
    P = ora.project(h64, ang, nd)
    S = 0.0
    for a in range(na):
        S += ora.curve_row(P[a], gamma * P[a], np.zeros(nd), flat[0, 0], flat[0, 1], flat[0, 2], mask,
                           drift=float(drift[a]), z=z, s_exp=s_exp[0, a])["cost"]
    return S + lam * (h64 ** 2).sum()


@pytest.mark.parametrize("seed,gamma,lam,z", [(0, 5.0, 0.0, 1.0), (1, 5.0, 1e-2, 0.5), (2, 2.0, 0.0, 2.0)])
def test_h_gradient_matches_finite_differences(seed, gamma, lam, z):
    ang, maps, flat, mask, drift, s_exp = tiny_problem(seed)
    h = maps[0]
    cost, grad, st = ora.cost_grad_h(ang, h, gamma, flat, mask, drift, s_exp, lam, z=z)
    h64 = h[0].astype(np.float64)
    c0 = _cost64(ang, h64, gamma, flat, mask, drift, s_exp, lam, z)
    assert abs(c0 - cost[0]) <= 1e-12 * abs(c0)
    step = 1e-4 * np.abs(h64).max()
    fd = np.zeros_like(h64)
    for idx in np.ndindex(*h64.shape):
        hp, hm = h64.copy(), h64.copy()
        hp[idx] += step
        hm[idx] -= step
        fd[idx] = (_cost64(ang, hp, gamma, flat, mask, drift, s_exp, lam, z) -
                   _cost64(ang, hm, gamma, flat, mask, drift, s_exp, lam, z)) / (2 * step)
    assert np.linalg.norm(fd - grad[0]) / np.linalg.norm(grad[0]) < 1e-6
    assert list(st) == [0, 0]


@pytest.mark.parametrize("seed,gamma", [(3, 5.0), (4, 0.7)])
def test_h_model_is_three_map_model_at_h_gamma_h_zero(seed, gamma):
    ang, maps, flat, mask, drift, s_exp = tiny_problem(seed, n=8, na=7, nd=13, m=1)
    h = maps[0]
    cost, grad, _ = ora.cost_grad_h(ang, h, gamma, flat, mask, drift, s_exp, 1e-2)
    mu, delta, sigma = h, (gamma * h.astype(np.float64)).astype(np.float32), np.zeros_like(h)
    # delta = gamma h rounded to fp32 for the three-map oracle: compare against its own fp64 input
    c3, gm, gd, gs, _ = ora.cost_grad(ang, mu, delta, sigma, flat, mask, drift, s_exp, 0.0)
    reg = 1e-2 * (h.astype(np.float64) ** 2).sum()
    assert abs(cost[0] - (c3[0] + reg)) <= 1e-6 * cost[0]          # fp32 rounding of gamma h only
    g_chain = gm[0] + gamma * gd[0] + 2e-2 * h[0].astype(np.float64)
    assert np.linalg.norm(grad[0] - g_chain) / np.linalg.norm(g_chain) < 1e-5


def test_gamma_zero_is_attenuation_times_flat():
    ang, maps, flat, mask, drift, _ = tiny_problem(5, n=8, na=6, nd=12, m=5)
    h = maps[0]
    smod = ora.cost_grad_h(ang, h, 0.0, flat, mask, drift)
    P = ora.project(h[0].astype(np.float64), ang, 12)
    A, c, w = (flat[0, q].astype(np.float64) for q in range(3))
    for a in range(len(ang)):
        for j, mj in enumerate(mask.astype(np.float64)):
            f = A * np.exp(-(mj - c - float(drift[a])) ** 2 / (2 * w * w))
            np.testing.assert_allclose(smod[0, a, j], np.exp(-P[a]) * f, rtol=1e-14, atol=0)


def test_h_exact_fit():
    ang, maps, flat, mask, drift, _ = tiny_problem(6, n=8, na=7, nd=13, m=1)
    h = maps[0]
    smod = ora.cost_grad_h(ang, h, 5.0, flat, mask, drift)
    s_exp = smod.astype(np.float32)
    bound = ((np.spacing(s_exp).astype(np.float64) / 2) ** 2).sum()
    cost, grad, _ = ora.cost_grad_h(ang, h, 5.0, flat, mask, drift, s_exp, 0.0)
    assert cost[0] <= bound
    c0, g0, _ = ora.cost_grad_h(ang, np.zeros_like(h), 5.0, flat, mask, drift, s_exp, 0.0)
    assert np.abs(grad).max() < 1e-6 * np.abs(g0).max()
