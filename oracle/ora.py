"""fp64 CPU oracle for the EI cost+gradient hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  It shares no code with the CUDA path
(``paper_2202_08627_b200``) and imports nothing from it.  The arithmetic lives in
``oracle/ora.c`` (plain fp64 loops, cited there line by line against PAPER.md / SPEC.md);
this file only builds that library and marshals numpy arrays.

Functions (fp64 unless noted; slices are independent):
  project(img, angles, n_det, dx, du)           a1, eq. 1
  backproject(sino, angles, n, dx, du)          a5, exact transpose
  diff_t / diff_t_adjoint                       a2
  curve_row(...)                                a2-a4 for one detector row (eq. 2, 4, 5)
  forward(geom, angles, mu, delta, sigma, flat, mask, drift)        -> s_mod [S][Na][M][Nd]
  cost_grad(geom, angles, ..., s_exp, lam)      -> cost[S], g_mu, g_delta, g_sigma, status
  cost_grad_h(angles, h, gamma, ...)            NEXT-3: the paper's single-map model, eq. 4
  ic_eval / cost_grad_hs(...)                   NEXT-4: sampled flat IC (periodic Catmull-Rom)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ora.c")
_LIB = os.path.join(_HERE, "libora.so")
_lib = None

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_fp = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile ora.c -> libora.so (gcc -O2 -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i, d = ctypes.c_int, ctypes.c_double
        L.ora_project.argtypes = [i, i, i, d, d, _dp, _dp, _dp]
        L.ora_backproject.argtypes = [i, i, i, d, d, _dp, _dp, _dp]
        L.ora_diff_t.argtypes = [i, d, _dp, _dp]
        L.ora_diff_t_adjoint.argtypes = [i, d, _dp, _dp]
        vp = ctypes.c_void_p
        L.ora_curve_row.argtypes = [i, i, d, d, _dp, _dp, _dp, _dp, _dp, _dp, _dp, d,
                                    vp, vp, vp, vp, vp, vp, _ip, vp]
        L.ora_forward.argtypes = [i, i, i, i, d, d, d, _dp, _fp, _fp, _fp, _fp, _fp, vp, _dp, _ip]
        L.ora_cost_grad.argtypes = [i, i, i, i, d, d, d, _dp, _fp, _fp, _fp, _fp, _fp, vp, _fp, d,
                                    vp, _dp, _dp, _dp, _ip]
        L.ora_cost_grad2.argtypes = L.ora_cost_grad.argtypes + [vp]
        L.ora_cost_grad_h.argtypes = [i, i, i, i, d, d, d, d, _dp, _fp, _fp, _fp, vp, vp, d, vp, vp, vp, _ip]
        L.ora_ic_eval.argtypes = [_fp, i, i, i, d, vp, vp]
        L.ora_cost_grad_hs.argtypes = [i, i, i, i, i, d, d, d, d, _dp, _fp, _fp, _fp, vp, vp, d, vp, vp, vp,
                                       _ip]
        L.ora_num_threads.restype = i
        _lib = L
    return _lib


def num_threads() -> int:
    return lib().ora_num_threads()


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def project(img, angles, n_det, dx=1.0, du=1.0):
    img, angles = _d(img), _d(angles)
    n = img.shape[-1]
    assert img.shape == (n, n)
    out = np.zeros((len(angles), n_det), np.float64)
    lib().ora_project(n, len(angles), n_det, dx, du, angles, img, out)
    return out


def backproject(sino, angles, n, dx=1.0, du=1.0):
    sino, angles = _d(sino), _d(angles)
    na, nd = sino.shape
    assert na == len(angles)
    out = np.zeros((n, n), np.float64)
    lib().ora_backproject(n, na, nd, dx, du, angles, sino, out)
    return out


def diff_t(p, du=1.0):
    p = _d(p)
    out = np.zeros_like(p)
    lib().ora_diff_t(len(p), du, p, out)
    return out


def diff_t_adjoint(g, du=1.0):
    g = _d(g)
    out = np.zeros_like(g)
    lib().ora_diff_t_adjoint(len(g), du, g, out)
    return out


def curve_row(p_mu, p_delta, p_sigma, flat_A, flat_c, flat_w, mask, drift=0.0, z=1.0, du=1.0,
              s_exp=None):
    """One detector row: returns dict(s_mod [M][Nd], and if s_exp: cost, g_mu, g_delta, g_sigma,
    g_drift = dS/dm_o, counters=[mu_clamp, w2_clamp])."""
    p_mu, p_delta, p_sigma = _d(p_mu), _d(p_delta), _d(p_sigma)
    fa, fc, fw, mk = _d(flat_A), _d(flat_c), _d(flat_w), _d(mask)
    nd, m = len(p_mu), len(mk)
    s_mod = np.zeros((m, nd), np.float64)
    cnt = np.zeros(2, np.int64)
    out = {"s_mod": s_mod}
    if s_exp is not None:
        se = _d(s_exp).reshape(m, nd)
        cost = np.zeros(1, np.float64)
        gm, gd, gs = (np.zeros(nd, np.float64) for _ in range(3))
        gmo = np.zeros(1, np.float64)
        lib().ora_curve_row(nd, m, du, z, p_mu, p_delta, p_sigma, fa, fc, fw, mk, float(drift),
                            _ptr(se), _ptr(s_mod), _ptr(cost), _ptr(gm), _ptr(gd), _ptr(gs), cnt,
                            _ptr(gmo))
        out.update(cost=float(cost[0]), g_mu=gm, g_delta=gd, g_sigma=gs, g_drift=float(gmo[0]))
    else:
        lib().ora_curve_row(nd, m, du, z, p_mu, p_delta, p_sigma, fa, fc, fw, mk, float(drift),
                            None, _ptr(s_mod), None, None, None, None, cnt, None)
    out["counters"] = cnt
    return out


def forward(angles, mu, delta, sigma, flat, mask, drift=None, n_det=None, dx=1.0, du=1.0, z=1.0):
    """s_mod [S][Na][M][Nd] (fp64) for fp32 inputs mu/delta/sigma [S][N][N], flat [S][3][Nd]."""
    angles = _d(angles)
    mu, delta, sigma, flat, mask = _f(mu), _f(delta), _f(sigma), _f(flat), _f(mask)
    S, n, _ = mu.shape
    nd = flat.shape[-1] if n_det is None else n_det
    na, m = len(angles), len(mask)
    dr = None if drift is None else _f(drift)
    out = np.zeros((S, na, m, nd), np.float64)
    cnt = np.zeros(2, np.int64)
    for s in range(S):
        o = np.zeros((na, m, nd), np.float64)
        lib().ora_forward(n, na, nd, m, dx, du, z, angles, mu[s], delta[s], sigma[s], flat[s], mask,
                          _ptr(dr), o, cnt)
        out[s] = o
    return out, cnt


def cost_grad(angles, mu, delta, sigma, flat, mask, drift, s_exp, lam=0.0, dx=1.0, du=1.0, z=1.0,
              slices=None, want_drift=False):
    """Per-slice cost (fp64) and gradient maps (fp64) of eq. 5; status [3] int64.
    want_drift: also return g_drift [S][Na] = dS_s/dm_o(theta) (NEXT-2) as a 6th value."""
    angles = _d(angles)
    mu, delta, sigma, flat, mask, s_exp = (_f(a) for a in (mu, delta, sigma, flat, mask, s_exp))
    S, n, _ = mu.shape
    na, m, nd = s_exp.shape[1:]
    dr = None if drift is None else _f(drift)
    sl = range(S) if slices is None else list(slices)
    cost = np.zeros(len(sl), np.float64)
    g = np.zeros((3, len(sl), n, n), np.float64)
    status = np.zeros(3, np.int64)
    gdr = np.zeros((len(sl), na), np.float64)
    for o, s in enumerate(sl):
        c = np.zeros(1, np.float64)
        gm, gd, gs = (np.zeros((n, n), np.float64) for _ in range(3))
        gmo = np.zeros(na, np.float64)
        lib().ora_cost_grad2(n, na, nd, m, dx, du, z, angles, mu[s], delta[s], sigma[s], flat[s], mask,
                             _ptr(dr), s_exp[s], float(lam), _ptr(c), gm, gd, gs, status, _ptr(gmo))
        cost[o] = c[0]
        g[0, o], g[1, o], g[2, o] = gm, gd, gs
        gdr[o] = gmo
    if want_drift:
        return cost, g[0], g[1], g[2], status, gdr
    return cost, g[0], g[1], g[2], status


def cost_grad_h(angles, h, gamma, flat, mask, drift, s_exp=None, lam=0.0, dx=1.0, du=1.0, z=1.0,
                want_smod=False):
    """The paper's single-map model (eq. 4, mu = gamma^-1 delta = h): per-slice cost (fp64),
    gradient map (fp64) and status [2] = (non-finite inputs, clamp hits); s_exp=None: forward only
    (returns s_mod [S][Na][M][Nd]).  With want_smod the s_mod array is appended."""
    angles = _d(angles)
    h, flat, mask = _f(h), _f(flat), _f(mask)
    S, n, _ = h.shape
    na = len(angles)
    m = len(mask)
    nd = flat.shape[-1]
    dr = None if drift is None else _f(drift)
    se = None if s_exp is None else _f(s_exp)
    cost = np.zeros(S)
    grad = np.zeros((S, n, n))
    smod = np.zeros((S, na, m, nd))
    status = np.zeros(2, np.int64)
    for s in range(S):
        c = np.zeros(1)
        g = np.zeros((n, n))
        sm = np.zeros((na, m, nd))
        lib().ora_cost_grad_h(n, na, nd, m, dx, du, z, float(gamma), angles, h[s], flat[s], mask,
                              _ptr(dr), None if se is None else _ptr(se[s]), float(lam), _ptr(c),
                              _ptr(g), _ptr(sm), status)
        cost[s], grad[s], smod[s] = c[0], g, sm
    if s_exp is None:
        return smod
    return (cost, grad, status, smod) if want_smod else (cost, grad, status)


def ic_eval(fs, t, m):
    """Sampled flat IC fs [K][Nd] at pixel t and mask position m (periods): (f, f')."""
    fs = _f(fs)
    K, nd = fs.shape
    f, fp = np.zeros(1), np.zeros(1)
    lib().ora_ic_eval(fs, K, nd, int(t), float(m), _ptr(f), _ptr(fp))
    return float(f[0]), float(fp[0])


def cost_grad_hs(angles, h, gamma, fs, mask, drift, s_exp=None, lam=0.0, dx=1.0, du=1.0, z=1.0):
    """Single-map model with the sampled flat IC fs [S][K][Nd] (NEXT-4).  s_exp=None: returns
    s_mod [S][Na][M][Nd]; else (cost [S], grad [S][N][N], status [2])."""
    angles = _d(angles)
    h, fs, mask = _f(h), _f(fs), _f(mask)
    S, n, _ = h.shape
    na, m = len(angles), len(mask)
    K, nd = fs.shape[1:]
    dr = None if drift is None else _f(drift)
    se = None if s_exp is None else _f(s_exp)
    cost, grad = np.zeros(S), np.zeros((S, n, n))
    smod = np.zeros((S, na, m, nd))
    status = np.zeros(2, np.int64)
    for s in range(S):
        c, g, sm = np.zeros(1), np.zeros((n, n)), np.zeros((na, m, nd))
        lib().ora_cost_grad_hs(n, na, nd, m, K, dx, du, z, float(gamma), angles, h[s], fs[s], mask,
                               _ptr(dr), None if se is None else _ptr(se[s]), float(lam), _ptr(c),
                               _ptr(g), _ptr(sm), status)
        cost[s], grad[s], smod[s] = c[0], g, sm
    if s_exp is None:
        return smod
    return cost, grad, status
