"""Thin Python binding of libei (include/ei.h).  Argument marshalling only: every numeric
step of the path runs in the CUDA kernels behind the C ABI.  There is no CPU fallback — if
libei.so is missing or cannot be loaded this module raises at import.

Device entry points take CUDA torch tensors (fp32, contiguous) and run asynchronously on
the current torch stream (or the stream passed in); ``ei_cost_grad_host`` takes numpy arrays.
Names and argument order follow the C functions.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libei.so")

if not os.path.exists(LIB_PATH):
    raise ImportError("libei.so not built (run `python -m paper_2202_08627_b200.build`); "
                      "the EI hot path has no CPU fallback")
_lib = ctypes.CDLL(LIB_PATH)

EI_OK, EI_ERR_NULL, EI_ERR_SHAPE, EI_ERR_DOMAIN, EI_ERR_RESOURCE, EI_ERR_CUDA = range(6)
SYMBOLS = ("ei_plan_create", "ei_plan_destroy", "ei_project", "ei_backproject", "ei_forward",
           "ei_cost_grad", "ei_cost_grad_drift", "ei_forward_h", "ei_cost_grad_h", "ei_forward_hs",
           "ei_cost_grad_hs", "ei_cost_grad_host", "ei_plan_stats", "ei_plan_set_timing",
           "ei_plan_read_timing", "ei_plan_info", "ei_error_string", "ei_version")
KERNELS = ("K0_pack", "K1_project", "K2_curve", "K3_backproject", "unused4", "unused5")


class ei_geometry(ctypes.Structure):
    _fields_ = [("n_slices", ctypes.c_int32), ("n", ctypes.c_int32), ("n_angles", ctypes.c_int32),
                ("n_det", ctypes.c_int32), ("n_mask", ctypes.c_int32), ("pixel", ctypes.c_double),
                ("det_pitch", ctypes.c_double), ("z", ctypes.c_double)]


_vp, _i, _f = ctypes.c_void_p, ctypes.c_int, ctypes.c_float
_lib.ei_plan_create.argtypes = [ctypes.POINTER(ei_geometry), _vp, ctypes.POINTER(_vp)]
_lib.ei_plan_destroy.argtypes = [_vp]
_lib.ei_plan_destroy.restype = None
_lib.ei_project.argtypes = [_vp, _vp, _i, _vp, _vp]
_lib.ei_backproject.argtypes = [_vp, _vp, _i, _vp, _vp]
_lib.ei_forward.argtypes = [_vp] + [_vp] * 7 + [_vp]
_lib.ei_cost_grad.argtypes = [_vp] + [_vp] * 7 + [_f] + [_vp] * 5 + [_vp]
_lib.ei_cost_grad_drift.argtypes = [_vp] + [_vp] * 7 + [_f] + [_vp] * 6 + [_vp]
_lib.ei_forward_h.argtypes = [_vp, _vp, _f] + [_vp] * 4 + [_vp]
_lib.ei_cost_grad_h.argtypes = [_vp, _vp, _f] + [_vp] * 4 + [_f] + [_vp] * 4 + [_vp]
_lib.ei_forward_hs.argtypes = [_vp, _vp, _f, _vp, _i] + [_vp] * 3 + [_vp]
_lib.ei_cost_grad_hs.argtypes = [_vp, _vp, _f, _vp, _i] + [_vp] * 3 + [_f] + [_vp] * 4 + [_vp]
_lib.ei_cost_grad_host.argtypes = [_vp] + [_vp] * 7 + [_f] + [_vp] * 5 + [_vp]
_lib.ei_plan_stats.argtypes = [_vp, _vp]
_lib.ei_plan_set_timing.argtypes = [_vp, _i]
_lib.ei_plan_info.argtypes = [_vp, _vp]
_lib.ei_plan_read_timing.argtypes = [_vp, _vp, _vp]
_lib.ei_error_string.argtypes = [_i]
_lib.ei_error_string.restype = ctypes.c_char_p
_lib.ei_version.restype = ctypes.c_char_p


class EIError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__("%s: %s (code %d)" % (where, ei_error_string(code), code))
        self.code = code


def ei_error_string(code: int) -> str:
    return _lib.ei_error_string(int(code)).decode()


def ei_version() -> str:
    return _lib.ei_version().decode()


def _check(rc: int, where: str):
    if rc != EI_OK:
        raise EIError(rc, where)


class Plan:
    """Owns an ei_plan*.  Geometry fields follow ei_geometry."""

    def __init__(self, n_slices, n, n_angles, n_det, n_mask, pixel, det_pitch, z, angles):
        self.geom = ei_geometry(int(n_slices), int(n), int(n_angles), int(n_det), int(n_mask),
                                float(pixel), float(det_pitch), float(z))
        self.angles = np.ascontiguousarray(angles, dtype=np.float64)
        if len(self.angles) != n_angles:
            raise ValueError("len(angles) != n_angles")
        h = _vp()
        _check(_lib.ei_plan_create(ctypes.byref(self.geom), self.angles.ctypes.data, ctypes.byref(h)),
               "ei_plan_create")
        self._h = h

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("plan destroyed")
        return self._h

    def destroy(self):
        if getattr(self, "_h", None) is not None:
            _lib.ei_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    @property
    def shape(self):
        g = self.geom
        return g.n_slices, g.n, g.n_angles, g.n_det, g.n_mask


def ei_plan_create(n_slices, n, n_angles, n_det, n_mask, pixel, det_pitch, z, angles) -> Plan:
    return Plan(n_slices, n, n_angles, n_det, n_mask, pixel, det_pitch, z, angles)


def ei_plan_destroy(plan: Plan):
    plan.destroy()


def ei_plan_stats(plan: Plan):
    out = (ctypes.c_int64 * 6)()
    _check(_lib.ei_plan_stats(plan.handle, out), "ei_plan_stats")
    return list(out)


def ei_plan_info(plan: Plan) -> dict:
    out = (ctypes.c_int64 * 12)()
    _check(_lib.ei_plan_info(plan.handle, out), "ei_plan_info")
    keys = ("k1_groups", "k1_rows_per_chunk", "k1_window", "k1_row_split", "window_overflows",
            "k1_smem_bytes", "k1_ray_fast", "k3_angle_split", "mirror_pairs", "k2_segments",
            "k1_band_rows", "k1_ctas")
    return dict(zip(keys, list(out)))


def ei_plan_set_timing(plan: Plan, max_evals: int):
    _check(_lib.ei_plan_set_timing(plan.handle, int(max_evals)), "ei_plan_set_timing")


def ei_plan_read_timing(plan: Plan):
    """-> (dict kernel -> summed ms, number of recorded evaluations)"""
    ms = (ctypes.c_double * 6)()
    n = ctypes.c_int()
    _check(_lib.ei_plan_read_timing(plan.handle, ms, ctypes.byref(n)), "ei_plan_read_timing")
    return dict(zip(KERNELS, list(ms))), n.value


# ---- tensor marshalling ---------------------------------------------------------------------
def _dev(t, shape: Sequence[int], name: str, dtype=None):
    import torch
    dtype = dtype or torch.float32
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("%s must be a CUDA tensor" % name)
    if t.dtype != dtype or not t.is_contiguous():
        raise TypeError("%s must be contiguous %s" % (name, dtype))
    if tuple(t.shape) != tuple(shape):
        raise ValueError("%s has shape %s, expected %s" % (name, tuple(t.shape), tuple(shape)))
    return t.data_ptr()


def _stream(stream):
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def ei_project(plan: Plan, maps, n_maps: int, sino, stream=None):
    S, N, NA, ND, _ = plan.shape
    _check(_lib.ei_project(plan.handle, _dev(maps, (S, n_maps, N, N), "maps"), int(n_maps),
                           _dev(sino, (S, n_maps, NA, ND), "sino"), _stream(stream)), "ei_project")


def ei_backproject(plan: Plan, sino, n_maps: int, maps, stream=None):
    S, N, NA, ND, _ = plan.shape
    _check(_lib.ei_backproject(plan.handle, _dev(sino, (S, n_maps, NA, ND), "sino"), int(n_maps),
                               _dev(maps, (S, n_maps, N, N), "maps"), _stream(stream)),
           "ei_backproject")


def ei_forward(plan: Plan, mu, delta, sigma, flat, mask_pos, drift, s_mod, stream=None):
    S, N, NA, ND, M = plan.shape
    _check(_lib.ei_forward(plan.handle, _dev(mu, (S, N, N), "mu"), _dev(delta, (S, N, N), "delta"),
                           _dev(sigma, (S, N, N), "sigma"), _dev(flat, (S, 3, ND), "flat"),
                           _dev(mask_pos, (M,), "mask_pos"),
                           None if drift is None else _dev(drift, (NA,), "drift"),
                           _dev(s_mod, (S, NA, M, ND), "s_mod"), _stream(stream)), "ei_forward")


def ei_cost_grad(plan: Plan, mu, delta, sigma, flat, mask_pos, drift, s_exp, lam: float, cost,
                 g_mu, g_delta, g_sigma, status, stream=None):
    import torch
    S, N, NA, ND, M = plan.shape
    _check(_lib.ei_cost_grad(
        plan.handle, _dev(mu, (S, N, N), "mu"), _dev(delta, (S, N, N), "delta"),
        _dev(sigma, (S, N, N), "sigma"), _dev(flat, (S, 3, ND), "flat"),
        _dev(mask_pos, (M,), "mask_pos"), None if drift is None else _dev(drift, (NA,), "drift"),
        _dev(s_exp, (S, NA, M, ND), "s_exp"), float(lam), _dev(cost, (S,), "cost", torch.float64),
        _dev(g_mu, (S, N, N), "g_mu"), _dev(g_delta, (S, N, N), "g_delta"),
        _dev(g_sigma, (S, N, N), "g_sigma"), _dev(status, (4,), "status", torch.int32),
        _stream(stream)), "ei_cost_grad")


def ei_cost_grad_drift(plan: Plan, mu, delta, sigma, flat, mask_pos, drift, s_exp, lam: float, cost,
                       g_mu, g_delta, g_sigma, g_drift, status, stream=None):
    """ei_cost_grad + g_drift [S][N_theta] = dS_s/dm_o(theta) (NEXT-2), same pass."""
    import torch
    S, N, NA, ND, M = plan.shape
    _check(_lib.ei_cost_grad_drift(
        plan.handle, _dev(mu, (S, N, N), "mu"), _dev(delta, (S, N, N), "delta"),
        _dev(sigma, (S, N, N), "sigma"), _dev(flat, (S, 3, ND), "flat"),
        _dev(mask_pos, (M,), "mask_pos"), None if drift is None else _dev(drift, (NA,), "drift"),
        _dev(s_exp, (S, NA, M, ND), "s_exp"), float(lam), _dev(cost, (S,), "cost", torch.float64),
        _dev(g_mu, (S, N, N), "g_mu"), _dev(g_delta, (S, N, N), "g_delta"),
        _dev(g_sigma, (S, N, N), "g_sigma"), _dev(g_drift, (S, NA), "g_drift"),
        _dev(status, (4,), "status", torch.int32), _stream(stream)), "ei_cost_grad_drift")


def ei_forward_h(plan: Plan, h, gamma: float, flat, mask_pos, drift, s_mod, stream=None):
    """Single-map model (NEXT-3, eq. 4 with mu = gamma^-1 delta = h): s_mod [S][N_theta][M][N_d]."""
    S, N, NA, ND, M = plan.shape
    _check(_lib.ei_forward_h(plan.handle, _dev(h, (S, N, N), "h"), float(gamma),
                             _dev(flat, (S, 3, ND), "flat"), _dev(mask_pos, (M,), "mask_pos"),
                             None if drift is None else _dev(drift, (NA,), "drift"),
                             _dev(s_mod, (S, NA, M, ND), "s_mod"), _stream(stream)), "ei_forward_h")


def ei_cost_grad_h(plan: Plan, h, gamma: float, flat, mask_pos, drift, s_exp, lam: float, cost, g_h,
                   g_drift, status, stream=None):
    """Single-map model (NEXT-3): cost [S] fp64, g_h [S][N][N], optional g_drift [S][N_theta]."""
    import torch
    S, N, NA, ND, M = plan.shape
    _check(_lib.ei_cost_grad_h(
        plan.handle, _dev(h, (S, N, N), "h"), float(gamma), _dev(flat, (S, 3, ND), "flat"),
        _dev(mask_pos, (M,), "mask_pos"), None if drift is None else _dev(drift, (NA,), "drift"),
        _dev(s_exp, (S, NA, M, ND), "s_exp"), float(lam), _dev(cost, (S,), "cost", torch.float64),
        _dev(g_h, (S, N, N), "g_h"), None if g_drift is None else _dev(g_drift, (S, NA), "g_drift"),
        _dev(status, (4,), "status", torch.int32), _stream(stream)), "ei_cost_grad_h")


def ei_forward_hs(plan: Plan, h, gamma: float, flat_samples, mask_pos, drift, s_mod, stream=None):
    """Single-map model with the sampled flat IC flat_samples [S][K][N_d] (NEXT-4)."""
    S, N, NA, ND, M = plan.shape
    K = int(flat_samples.shape[1])
    _check(_lib.ei_forward_hs(plan.handle, _dev(h, (S, N, N), "h"), float(gamma),
                              _dev(flat_samples, (S, K, ND), "flat_samples"), K,
                              _dev(mask_pos, (M,), "mask_pos"),
                              None if drift is None else _dev(drift, (NA,), "drift"),
                              _dev(s_mod, (S, NA, M, ND), "s_mod"), _stream(stream)), "ei_forward_hs")


def ei_cost_grad_hs(plan: Plan, h, gamma: float, flat_samples, mask_pos, drift, s_exp, lam: float, cost,
                    g_h, g_drift, status, stream=None):
    """Single-map model with the sampled flat IC (NEXT-4): cost, g_h, optional g_drift."""
    import torch
    S, N, NA, ND, M = plan.shape
    K = int(flat_samples.shape[1])
    _check(_lib.ei_cost_grad_hs(
        plan.handle, _dev(h, (S, N, N), "h"), float(gamma), _dev(flat_samples, (S, K, ND), "flat_samples"),
        K, _dev(mask_pos, (M,), "mask_pos"), None if drift is None else _dev(drift, (NA,), "drift"),
        _dev(s_exp, (S, NA, M, ND), "s_exp"), float(lam), _dev(cost, (S,), "cost", torch.float64),
        _dev(g_h, (S, N, N), "g_h"), None if g_drift is None else _dev(g_drift, (S, NA), "g_drift"),
        _dev(status, (4,), "status", torch.int32), _stream(stream)), "ei_cost_grad_hs")


def _host(a, shape, name, dtype=np.float32, writable=False):
    if not isinstance(a, np.ndarray) or a.dtype != dtype or not a.flags.c_contiguous:
        raise TypeError("%s must be a C-contiguous numpy %s array" % (name, np.dtype(dtype)))
    if tuple(a.shape) != tuple(shape):
        raise ValueError("%s has shape %s, expected %s" % (name, a.shape, tuple(shape)))
    if writable and not a.flags.writeable:
        raise ValueError("%s must be writable" % name)
    return a.ctypes.data


def ei_cost_grad_host(plan: Plan, mu, delta, sigma, flat, mask_pos, drift, s_exp, lam: float,
                      cost, g_mu, g_delta, g_sigma, status, stream=None):
    """Host-buffer variant: numpy inputs/outputs (pinned memory recommended)."""
    S, N, NA, ND, M = plan.shape
    _check(_lib.ei_cost_grad_host(
        plan.handle, _host(mu, (S, N, N), "mu"), _host(delta, (S, N, N), "delta"),
        _host(sigma, (S, N, N), "sigma"), _host(flat, (S, 3, ND), "flat"),
        _host(mask_pos, (M,), "mask_pos"), None if drift is None else _host(drift, (NA,), "drift"),
        _host(s_exp, (S, NA, M, ND), "s_exp"), float(lam),
        _host(cost, (S,), "cost", np.float64, True), _host(g_mu, (S, N, N), "g_mu", writable=True),
        _host(g_delta, (S, N, N), "g_delta", writable=True),
        _host(g_sigma, (S, N, N), "g_sigma", writable=True),
        _host(status, (4,), "status", np.int32, True), _stream(stream)), "ei_cost_grad_host")


# ---- allocating conveniences (same kernels) -------------------------------------------------
class Workspace:
    """Output tensors for repeated ei_cost_grad calls on one plan (no per-call allocation)."""

    def __init__(self, plan: Plan, device="cuda"):
        import torch
        S, N, NA, ND, M = plan.shape
        self.cost = torch.zeros(S, dtype=torch.float64, device=device)
        self.g = torch.zeros(3, S, N, N, dtype=torch.float32, device=device)
        self.status = torch.zeros(4, dtype=torch.int32, device=device)
        self.g_drift = torch.zeros(S, NA, dtype=torch.float32, device=device)


def cost_grad(plan: Plan, maps, flat, mask_pos, drift, s_exp, lam: float = 0.0,
              ws: Optional[Workspace] = None, stream=None, want_drift: bool = False):
    """Returns (cost [S] fp64, (g_mu, g_delta, g_sigma), status[4]) as device tensors;
    with want_drift a 4th value g_drift [S][N_theta] (ei_cost_grad_drift)."""
    ws = ws or Workspace(plan, maps[0].device)
    ws.status.zero_()
    if want_drift:
        ei_cost_grad_drift(plan, maps[0], maps[1], maps[2], flat, mask_pos, drift, s_exp, lam,
                           ws.cost, ws.g[0], ws.g[1], ws.g[2], ws.g_drift, ws.status, stream)
        return ws.cost, (ws.g[0], ws.g[1], ws.g[2]), ws.status, ws.g_drift
    ei_cost_grad(plan, maps[0], maps[1], maps[2], flat, mask_pos, drift, s_exp, lam, ws.cost,
                 ws.g[0], ws.g[1], ws.g[2], ws.status, stream)
    return ws.cost, (ws.g[0], ws.g[1], ws.g[2]), ws.status
