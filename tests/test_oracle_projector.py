"""Pins for the oracle's projector R_J, its transpose and D (CPU only, no GPU).

Each test checks the oracle against something other than itself: numpy sums (special
angles), textbook closed forms (Gaussian blob, ellipse chord, disk), an independently
written pixel-driven tent kernel, the adjoint identity and hand-derived golden values.
Citations: P:n = PAPER.md line, S:n = SPEC.md line, R# = DESIGN.md reading.
"""
import json
import os

import numpy as np
import pytest

from oracle import ora
from paper_2202_08627_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rel_l2(a, b):
    return np.linalg.norm(np.ravel(a - b)) / np.linalg.norm(np.ravel(b))


# ---- special angles: theta = 0, 90, 180, 270 deg reduce to numpy sums (R6, R7) ----------------
@pytest.mark.parametrize("n,nd", [(16, 22), (17, 23), (12, 12)])
def test_axis_angles_are_column_and_row_sums(n, nd):
    rng = np.random.default_rng(1)
    img = rng.uniform(size=(n, n))
    ang = np.deg2rad([0.0, 90.0, 180.0, 270.0])
    P = ora.project(img, ang, nd)
    off = (nd - n) // 2
    cols, rows = img.sum(axis=0), img.sum(axis=1)
    # theta=0: ray k sits at x = u_k -> integrates column j = k - off over y
    np.testing.assert_allclose(P[0, off:off + n], cols, rtol=1e-14, atol=1e-13)
    # theta=90: u = y -> row i = k - off
    np.testing.assert_allclose(P[1, off:off + n], rows, rtol=1e-14, atol=1e-13)
    # theta=180: u = -x -> reversed columns; theta=270: u = -y -> reversed rows
    np.testing.assert_allclose(P[2, off:off + n], cols[::-1], rtol=1e-14, atol=1e-13)
    np.testing.assert_allclose(P[3, off:off + n], rows[::-1], rtol=1e-14, atol=1e-13)
    outside = np.r_[0:off, off + n:nd]
    assert outside.size == 0 or np.abs(P[:, outside]).max() < 1e-13     # cos(270 deg) = -1.8e-16 leaks 1e-15-size weights


# ---- closed-form line integrals ------------------------------------------------------------
def _centred(n):
    return np.arange(n) - (n - 1) / 2.0


def test_gaussian_blob_closed_form():
    """Pixel-sampled Gaussian exp(-r^2/2s^2), s=N/12, off centre: its line integral is
    sqrt(2 pi) s exp(-(u-u0)^2 / 2s^2) with u0 = x0 cos + y0 sin (textbook).  Linear
    interpolation is second order, so the error must also fall ~4x per doubling of N."""
    errs = []
    for n in (64, 128, 256):
        s0, x0, y0 = n / 12.0, 0.06 * n, -0.04 * n
        x = _centred(n)[None, :]
        y = _centred(n)[:, None]
        img = np.exp(-((x - x0) ** 2 + (y - y0) ** 2) / (2 * s0 ** 2))
        nd = int(1.5 * n)
        ang = np.deg2rad(np.linspace(0, 360, 32, endpoint=False) + 0.3)
        ang = np.r_[ang, np.deg2rad([45.0, 135.0])]
        P = ora.project(img, ang, nd)
        u = _centred(nd)[None, :]
        u0 = (x0 * np.cos(ang) + y0 * np.sin(ang))[:, None]
        ref = np.sqrt(2 * np.pi) * s0 * np.exp(-(u - u0) ** 2 / (2 * s0 ** 2))
        errs.append(rel_l2(P, ref))
    assert errs[0] < 2.5e-3 and errs[1] < 6.5e-4 and errs[2] < 1.6e-4, errs
    for e0, e1 in zip(errs, errs[1:]):
        assert 3.5 < e0 / e1 < 4.5, errs


@pytest.mark.parametrize("n,tol", [(64, 4e-2), (128, 1.5e-2), (256, 1e-2)])
def test_ellipse_chord_closed_form(n, tol):
    """Sum of 8 random ellipses (R18) vs the textbook chord (2 rho a b / s^2) sqrt(s^2 - t^2),
    s^2 = a^2 cos^2(th-phi) + b^2 sin^2(th-phi)."""
    rng = np.random.default_rng(5)
    ell = synth.draw_ellipses(rng, n, 8)
    rho = rng.uniform(0.2, 1.0, 8)
    img = synth.raster(n, ell, rho)
    nd = int(1.5 * n)
    ang = np.deg2rad(np.linspace(0, 180, 24, endpoint=False) + 0.1)
    P = ora.project(img, ang, nd)
    u = _centred(nd)[None, :]
    ref = np.zeros_like(P)
    for (a, b, phi, x0, y0), r in zip(ell, rho):
        s2 = (a * np.cos(ang - phi)) ** 2 + (b * np.sin(ang - phi)) ** 2
        t = u - (x0 * np.cos(ang) + y0 * np.sin(ang))[:, None]
        ref += np.where(t ** 2 < s2[:, None], 2 * r * a * b / s2[:, None] *
                        np.sqrt(np.maximum(s2[:, None] - t ** 2, 0)), 0.0)
    assert rel_l2(P, ref) < tol


def test_spec_disk_chord():
    """centred disk radius R=N/4 (N=128): row at offset u ~ 2 sqrt(R^2-u^2), L2 err < 2 %,
    and all angles equal (rotation consistency < 1 %)."""
    n, R = 128, 32.0
    img = synth.raster(n, np.array([[R, R, 0.0, 0.0, 0.0]]), np.array([1.0]))
    ang = np.deg2rad(np.linspace(0, 180, 16, endpoint=False) + 0.7)
    P = ora.project(img, ang, n)
    u = _centred(n)
    ref = 2 * np.sqrt(np.maximum(R * R - u * u, 0))
    for row in P:
        assert rel_l2(row, ref) < 2e-2
    mean = P.mean(axis=0)
    for row in P:
        assert np.linalg.norm(row - mean) / np.linalg.norm(mean) < 1e-2


# ---- independent transpose: pixel-driven tent kernel --------------------
def tent_matrix(n, nd, ang, dx, du):
    """Dense B[(a,k),(i,j)] = (dx/|c_dom|) max(0, 1 - |k - k*|/h), k* = (x_j c + y_i s)/du +
    (Nd-1)/2, h = |c_dom| dx/du: the Joseph weight written pixel-first (no oracle code)."""
    x = _centred(n) * dx
    B = np.zeros((len(ang), nd, n, n))
    kk = np.arange(nd)[:, None, None]
    for a, th in enumerate(ang):
        c, s = np.cos(th), np.sin(th)
        cd = max(abs(c), abs(s))
        h = cd * dx / du
        kstar = (x[None, :] * c + x[:, None] * s) / du + (nd - 1) / 2.0
        B[a] = (dx / cd) * np.maximum(0.0, 1.0 - np.abs(kk - kstar[None]) / h)
    return B.reshape(len(ang) * nd, n * n)


@pytest.mark.parametrize("n,nd,span,dx,du", [(8, 12, 180, 1.0, 1.0), (9, 14, 360, 1.0, 1.0),
                                             (6, 11, 360, 0.8, 1.0), (7, 9, 180, 1.0, 1.3)])
def test_projector_equals_tent_kernel(n, nd, span, dx, du):
    ang = np.r_[np.deg2rad(np.linspace(0, span, 11, endpoint=False) + 0.37), np.pi / 4, 3 * np.pi / 4]
    A = np.zeros((len(ang) * nd, n * n))
    for p in range(n * n):
        e = np.zeros(n * n)
        e[p] = 1.0
        A[:, p] = ora.project(e.reshape(n, n), ang, nd, dx, du).ravel()
    B = tent_matrix(n, nd, ang, dx, du)
    assert np.abs(A - B).max() < 1e-12
    # the oracle's scatter is the transpose of its gather
    At = np.zeros((n * n, len(ang) * nd))
    for q in range(len(ang) * nd):
        e = np.zeros(len(ang) * nd)
        e[q] = 1.0
        At[:, q] = ora.backproject(e.reshape(len(ang), nd), ang, n, dx, du).ravel()
    assert np.abs(At - A.T).max() < 1e-14


def test_golden_tiny_projection():
    """Hand-derived values (tests/golden/tiny_projection.json, derivation inside)."""
    g = json.load(open(os.path.join(GOLDEN, "tiny_projection.json")))
    img = np.array(g["image"], float)
    for case in g["cases"]:
        P = ora.project(img, np.deg2rad([case["theta_deg"]]), g["n_det"])
        np.testing.assert_allclose(P[0], case["sinogram"], rtol=1e-14, atol=1e-14)


def test_linearity_zero_and_dot():
    rng = np.random.default_rng(3)
    n, nd = 24, 37
    ang = np.deg2rad(np.linspace(0, 360, 29, endpoint=False) + 0.2)
    assert np.all(ora.project(np.zeros((n, n)), ang, nd) == 0)
    x, y = rng.normal(size=(2, n, n))
    a, b = 1.7, -0.3
    lhs = ora.project(a * x + b * y, ang, nd)
    rhs = a * ora.project(x, ang, nd) + b * ora.project(y, ang, nd)
    assert rel_l2(lhs, rhs) < 1e-12
    for t in range(100):
        xi = rng.normal(size=(n, n))
        yi = rng.normal(size=(len(ang), nd))
        l = np.vdot(ora.project(xi, ang, nd), yi)
        r = np.vdot(xi, ora.backproject(yi, ang, n))
        assert abs(l - r) <= 1e-12 * max(abs(l), abs(r), 1e-300) * 10


# ---- D and D^T ---------------------------------------------------------------------
def test_diff_t_pins():
    nd = 256
    t = np.arange(nd, dtype=float)
    assert np.all(ora.diff_t(np.full(nd, 3.2)) == 0)
    np.testing.assert_allclose(ora.diff_t(2.5 * t - 1), 2.5, rtol=1e-14)      # exact on ramps
    k = 2 * np.pi / 64
    d = ora.diff_t(np.sin(k * t))
    err = np.abs(d[1:-1] - k * np.cos(k * t[1:-1])).max()
    assert err < k ** 3 / 6 * 1.01                                             # central O(k^3)
    rng = np.random.default_rng(0)
    for du in (1.0, 0.7):
        x, y = rng.normal(size=(2, 31))
        assert abs(np.dot(ora.diff_t(x, du), y) - np.dot(x, ora.diff_t_adjoint(y, du))) < 1e-12
    # D^T 1: column sums of D = [-3/2, +1/2, 0, ..., 0, -1/2, +3/2] (hand-derived)
    y = ora.diff_t_adjoint(np.ones(9))
    np.testing.assert_allclose(y, [-1.5, 0.5, 0, 0, 0, 0, 0, -0.5, 1.5], atol=1e-15)
