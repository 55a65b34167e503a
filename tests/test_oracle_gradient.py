"""Pins for the oracle's full cost and gradient (eq. 5) — CPU only.

* central finite differences of S on N <= 8 grids, all three maps, random drift, lambda in
  {0, 1e-2} (SURVEY.md CHECK-4)
* exact fit: s_exp = s_mod(truth) -> S and grad vanish up to the fp32 rounding of s_exp
  (S:267); with lambda > 0 the cost is lambda sum x^2
* slices are independent problems
"""
import numpy as np
import pytest

from oracle import ora


def tiny_problem(seed, n=6, na=5, nd=10, m=4, span=np.pi):
    rng = np.random.default_rng(seed)
    ang = np.arange(na) * span / na + 0.1
    mu = rng.uniform(0, 0.02, (1, n, n)).astype(np.float32)
    delta = rng.uniform(0, 0.02, (1, n, n)).astype(np.float32)
    sigma = rng.uniform(0, 2e-4, (1, n, n)).astype(np.float32)
    flat = np.stack([1e4 * (1 + rng.uniform(-0.05, 0.05, nd)), rng.normal(0, 0.05, nd),
                     0.15 * np.ones(nd)])[None].astype(np.float32)
    mask = np.linspace(-0.3, 0.3, m).astype(np.float32)
    drift = rng.normal(0, 0.01, na).astype(np.float32)
    s_exp = rng.uniform(0, 1.2e4, (1, na, m, nd)).astype(np.float32)
    return ang, [mu, delta, sigma], flat, mask, drift, s_exp


def _cost64(ang, maps64, flat, mask, drift, s_exp, lam, z):
    """Cost with fp64 map perturbations: the oracle takes fp32 maps, so evaluate via
    project + curve_row, which is the same arithmetic the oracle's cost uses."""
    na, m, nd = s_exp.shape[1:]
    P = [ora.project(x, ang, nd) for x in maps64]
    S = 0.0
    for a in range(na):
        S += ora.curve_row(P[0][a], P[1][a], P[2][a], flat[0, 0], flat[0, 1], flat[0, 2], mask,
                           drift=float(drift[a]), z=z, s_exp=s_exp[0, a])["cost"]
    return S + lam * sum((x ** 2).sum() for x in maps64)


@pytest.mark.parametrize("seed,lam,z,span", [(0, 0.0, 1.0, np.pi), (1, 1e-2, 2.0, 2 * np.pi),
                                             (2, 0.0, 0.5, np.pi)])
def test_gradient_matches_finite_differences(seed, lam, z, span):
    ang, maps, flat, mask, drift, s_exp = tiny_problem(seed, span=span)
    cost, gm, gd, gs, st = ora.cost_grad(ang, *maps, flat, mask, drift, s_exp, lam, z=z)
    maps64 = [x[0].astype(np.float64) for x in maps]
    c0 = _cost64(ang, maps64, flat, mask, drift, s_exp, lam, z)
    assert abs(c0 - cost[0]) <= 1e-12 * abs(c0)
    for q, g in enumerate((gm[0], gd[0], gs[0])):
        h = 1e-4 * np.abs(maps64[q]).max()
        fd = np.zeros_like(g)
        for idx in np.ndindex(*g.shape):
            xp = [x.copy() for x in maps64]
            xm = [x.copy() for x in maps64]
            xp[q][idx] += h
            xm[q][idx] -= h
            fd[idx] = (_cost64(ang, xp, flat, mask, drift, s_exp, lam, z) -
                       _cost64(ang, xm, flat, mask, drift, s_exp, lam, z)) / (2 * h)
        assert np.linalg.norm(fd - g) / np.linalg.norm(g) < 1e-6, (q, np.linalg.norm(fd - g) / np.linalg.norm(g))


def test_exact_fit_and_regulariser():
    ang, maps, flat, mask, drift, _ = tiny_problem(4, n=8, na=7, nd=13, m=5)
    smod, _ = ora.forward(ang, *maps, flat, mask, drift)
    s_exp = smod.astype(np.float32)
    # the only residual left is the fp32 rounding of s_exp: |r| <= ulp/2
    bound = ((np.spacing(s_exp.astype(np.float32)).astype(np.float64) / 2) ** 2).sum()
    cost, gm, gd, gs, st = ora.cost_grad(ang, *maps, flat, mask, drift, s_exp, 0.0)
    assert cost[0] <= bound
    zero = [np.zeros_like(x) for x in maps]
    c0, g0m, g0d, g0s, _ = ora.cost_grad(ang, *zero, flat, mask, drift, s_exp, 0.0)
    for g, gref in ((gm, g0m), (gs, g0s)):
        assert np.abs(g).max() < 1e-6 * np.abs(gref).max()
    lam = 1e-2
    reg = lam * sum((x.astype(np.float64) ** 2).sum() for x in maps)
    cost_l, gml, _, _, _ = ora.cost_grad(ang, *maps, flat, mask, drift, s_exp, lam)
    assert abs(cost_l[0] - reg) <= bound + 1e-14 * reg
    np.testing.assert_allclose(gml - gm, 2 * lam * maps[0].astype(np.float64), rtol=1e-12, atol=1e-13)


def test_slices_independent_and_status():
    a1 = tiny_problem(5)
    a2 = tiny_problem(6)
    stack = [np.concatenate([x, y]) for x, y in zip(a1[1], a2[1])]
    flat = np.concatenate([a1[2], a2[2]])
    s_exp = np.concatenate([a1[5], a2[5]])
    c, gm, gd, gs, st = ora.cost_grad(a1[0], *stack, flat, a1[3], a1[4], s_exp)
    c1, g1, _, _, _ = ora.cost_grad(a1[0], *a1[1], a1[2], a1[3], a1[4], a1[5])
    c2, g2, _, _, _ = ora.cost_grad(a1[0], *a2[1], a2[2], a1[3], a1[4], a2[5])
    assert c[0] == c1[0] and c[1] == c2[0]
    assert np.array_equal(gm[0], g1[0]) and np.array_equal(gm[1], g2[0])
    assert list(st) == [0, 0, 0]
    bad = [x.copy() for x in a1[1]]
    bad[1][0, 2, 3] = np.nan
    s_bad = a1[5].copy()
    s_bad[0, 0, 0, 0] = np.inf
    _, _, _, _, st = ora.cost_grad(a1[0], *bad, a1[2], a1[3], a1[4], s_bad)
    assert st[0] == 2


@pytest.mark.parametrize("seed,z", [(7, 1.0), (8, 2.5)])
def test_drift_gradient_matches_finite_differences(seed, z):
    """NEXT-2: dS/dm_o(theta) (m_o enters eq. 4, through u = m - c - m_o - Delta)
    against central differences of the fp64 cost in each drift component."""
    ang, maps, flat, mask, drift, s_exp = tiny_problem(seed)
    cost, gm, gd, gs, st, gdr = ora.cost_grad(ang, *maps, flat, mask, drift, s_exp, 0.0, z=z,
                                              want_drift=True)
    maps64 = [x[0].astype(np.float64) for x in maps]
    d64 = drift.astype(np.float64)
    h = 1e-5
    fd = np.zeros(len(d64))
    for a in range(len(d64)):
        dp, dm = d64.copy(), d64.copy()
        dp[a] += h
        dm[a] -= h
        fd[a] = (_cost64(ang, maps64, flat, mask, dp, s_exp, 0.0, z) -
                 _cost64(ang, maps64, flat, mask, dm, s_exp, 0.0, z)) / (2 * h)
    assert np.linalg.norm(fd - gdr[0]) / np.linalg.norm(gdr[0]) < 1e-6
    # a shift of every drift component by a is a shift of every mask position by -a (eq. 4):
    # sum_theta dS/dm_o = -sum_j dS/dm_j, checked by moving the mask instead
    mk = mask.astype(np.float64)
    cp = _cost64(ang, maps64, flat, mk - h, d64, s_exp, 0.0, z)
    cm = _cost64(ang, maps64, flat, mk + h, d64, s_exp, 0.0, z)
    assert abs((cp - cm) / (2 * h) - gdr[0].sum()) <= 1e-6 * np.abs(gdr[0]).sum()
