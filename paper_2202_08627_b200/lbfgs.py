"""Host L-BFGS loop driving `ei_cost_grad` (the paper minimises eq. 5 with
SciPy's L-BFGS, slice by slice).  Not the hot path: every cost and
gradient comes from one `ei_cost_grad` call; this module only does the optimizer's vector
arithmetic (torch ops on the device) and bookkeeping.

Design (stated here because the paper gives no optimizer parameters):
  * slices are independent problems: each slice keeps its own history, step length and
    convergence flag, but all slices are evaluated together in one batched call;
  * two-loop recursion (history m = 10) with a block-diagonal initial matrix: one scalar
    gamma per (slice, map) from the newest pair, gamma = <s_q, y_q> / <y_q, y_q>, because mu, delta
    and sigma differ by orders of magnitude and one scalar would precondition two of them badly;
  * batched backtracking Armijo line search (c1 = 1e-4, halving, <= 30 trials); a pair is
    stored only if <s, y> > 1e-12 |s| |y| (curvature), otherwise the history of that slice resets;
  * stop a slice when its relative cost decrease over an accepted step is below rel_tol, or when
    max_iter iterations are done.
Dot products: products in the iterate's dtype, sums in fp64.
"""
from __future__ import annotations

import dataclasses
import time
from typing import Callable, List, Optional, Tuple

import torch


@dataclasses.dataclass
class Result:
    x: torch.Tensor                 # [B, S, ...] final iterate (B = blocks, e.g. the 3 maps)
    cost: torch.Tensor              # [S] fp64 final cost
    history: List[torch.Tensor]     # per accepted iteration: [S] fp64 cost
    n_iter: int
    n_evals: int
    converged: torch.Tensor         # [S] bool
    seconds: float


def _bdot(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """Per-(block, slice) dot products, products in the tensors' dtype, sums in fp64: [B, S]."""
    B, S = a.shape[:2]
    return torch.sum(a.reshape(B, S, -1) * b.reshape(B, S, -1), dim=-1, dtype=torch.float64)


def _sdot(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """Per-slice dot products over all blocks: [S]."""
    return _bdot(a, b).sum(0)


def _bc(v: torch.Tensor, like: torch.Tensor) -> torch.Tensor:
    """Broadcast a [S] or [B, S] tensor against [B, S, ...]."""
    if v.dtype != torch.bool:
        v = v.to(like.dtype)
    if v.dim() == 1:
        v = v.unsqueeze(0)
    return v.reshape(v.shape + (1,) * (like.dim() - 2))


def minimize(fg: Callable[[torch.Tensor], Tuple[torch.Tensor, torch.Tensor]], x0: torch.Tensor,
             max_iter: int = 200, m: int = 10, rel_tol: float = 1e-9, c1: float = 1e-4,
             max_ls: int = 30, callback: Optional[Callable[[int, torch.Tensor], None]] = None) -> Result:
    """Minimise S independent problems.  x0: [B, S, ...]; fg(x) -> (cost [S] fp64, grad like x).

    The (s, y) history lives in two preallocated ring tensors [m, B, S, ...] with per-(pair,
    slice) rho = 1 / <s, y> (0 where the pair is not valid for that slice), so the two-loop
    recursion is a handful of fused tensor ops per pair instead of per-pair allocations."""
    t0 = time.time()
    x = x0.clone()
    f, g = fg(x)
    f, g = f.double().clone(), g.clone()
    n_evals = 1
    B, S = x.shape[:2]
    dev = x.device
    Sh = torch.zeros((m,) + tuple(x.shape), dtype=x.dtype, device=dev)
    Yh = torch.zeros_like(Sh)
    rho = torch.zeros(m, S, dtype=torch.float64, device=dev)
    nh, head = 0, 0                          # stored pairs, next ring slot
    gamma = torch.zeros(B, S, dtype=torch.float64, device=dev)   # block-diagonal initial scaling
    has_gamma = torch.zeros(S, dtype=torch.bool, device=dev)
    conv = torch.zeros(S, dtype=torch.bool, device=dev)
    sd = torch.ones(S, dtype=torch.bool, device=dev)   # current direction is steepest descent
    history = [f.clone()]
    it = 0
    for it in range(1, max_iter + 1):
        # ---- two-loop recursion: p = -H g (per slice, masked histories) ----
        q = g.clone()
        slots = [(head - nh + j) % m for j in range(nh)]     # oldest .. newest
        alphas = []
        for k in reversed(slots):
            a = rho[k] * _sdot(Sh[k], q)
            alphas.append(a)
            q.sub_(Yh[k] * _bc(a, q))
        # slices without a curvature pair yet: unit-length steepest-descent step per block
        gnorm = _bdot(g, g).sqrt().clamp_min(1e-300)
        scal = torch.where(has_gamma.unsqueeze(0), gamma, 1.0 / gnorm)
        r = q * _bc(scal, q)
        for k, a in zip(slots, reversed(alphas)):
            b = rho[k] * _sdot(Yh[k], r)
            r.add_(Sh[k] * _bc(a - b, r))
        p = -r
        gp = _sdot(g, p)
        bad = gp >= 0                          # not a descent direction: restart that slice
        # (masked updates instead of a host-side `if bad.any()`: no device -> host sync)
        p = torch.where(_bc(bad, p), -g * _bc(1.0 / gnorm, g), p)
        gp = torch.where(bad, _sdot(g, p), gp)
        rho = rho * (~bad).to(rho.dtype)
        sd = sd | bad
        # ---- batched backtracking Armijo ----
        step = torch.ones(S, dtype=torch.float64, device=dev)
        step = torch.where(conv, torch.zeros_like(step), step)
        accepted = conv.clone()
        x_new, f_new, g_new = x.clone(), f.clone(), g.clone()
        for _ in range(max_ls):
            xt = x + _bc(step, x) * p
            ft, gt = fg(xt)
            n_evals += 1
            ok = (~accepted) & (ft.double() <= f + c1 * step * gp)
            sel = _bc(ok, x)
            x_new = torch.where(sel, xt, x_new)
            g_new = torch.where(sel, gt, g_new)
            f_new = torch.where(ok, ft.double(), f_new)
            accepted |= ok
            if bool(accepted.all()):
                break
            step = torch.where(accepted, step, 0.5 * step)
        # no decrease found: restart that slice from steepest descent; if even that fails the
        # slice has converged to working precision
        failed = ~accepted
        rho = rho * accepted.to(rho.dtype)
        has_gamma = has_gamma & accepted
        s_vec, y_vec = x_new - x, g_new - g
        sy = _sdot(s_vec, y_vec)
        yy = _sdot(y_vec, y_vec)
        curv = sy > 1e-12 * _sdot(s_vec, s_vec).sqrt() * yy.sqrt()
        keep = accepted & curv & ~conv
        # the pair is stored for every slice (rho = 0 where it is not kept): no host-side branch
        Sh[head].copy_(s_vec)
        Yh[head].copy_(y_vec)
        rho[head] = torch.where(keep, 1.0 / sy.clamp_min(1e-300), torch.zeros_like(sy))
        head = (head + 1) % m
        nh = min(nh + 1, m)
        gb = _bdot(s_vec, y_vec) / _bdot(y_vec, y_vec).clamp_min(1e-300)
        gg = (sy / yy.clamp_min(1e-300)).unsqueeze(0).expand_as(gb)
        gb = torch.where(gb > 0, gb, gg)              # block secant not positive: global scalar
        gamma = torch.where(keep.unsqueeze(0), gb, gamma)
        has_gamma = has_gamma | keep
        rel = (f - f_new) / f.abs().clamp_min(1e-300)
        conv = conv | (failed & sd) | (accepted & (rel < rel_tol))
        sd = failed & ~conv
        x, f, g = x_new, f_new, g_new
        history.append(f.clone())
        if callback is not None:
            callback(it, f)
        if bool(conv.all()):
            break
    return Result(x, f, history, it, n_evals, conv, time.time() - t0)


def ei_objective(plan, flat, mask, drift, s_exp, lam: float = 1e-2, ws=None):
    """fg(x) for x = [3, S, N, N] (mu, delta, sigma) through the C ABI (`ei_cost_grad`)."""
    from . import ei
    ws = ws or ei.Workspace(plan, s_exp.device)

    def fg(x: torch.Tensor):
        x = x.contiguous()
        ws.status.zero_()
        ei.ei_cost_grad(plan, x[0], x[1], x[2], flat, mask, drift, s_exp, lam, ws.cost, ws.g[0], ws.g[1],
                        ws.g[2], ws.status)
        return ws.cost.clone(), ws.g.clone()
    return fg


def ei_objective_h(plan, gamma: float, flat, mask, drift, s_exp, lam: float = 1e-2,
                   flat_samples: bool = False):
    """fg(x) for x = [1, S, N, N] (the paper's single map h, eq. 4 with mu = gamma^-1 delta = h,
    PAPER.md:64) through `ei_cost_grad_h`, or `ei_cost_grad_hs` when `flat` holds the sampled flat
    IC [S][K][N_d] (flat_samples=True)."""
    from . import ei
    S, N, NA, ND, M = plan.shape
    cost = torch.zeros(S, dtype=torch.float64, device=s_exp.device)
    g = torch.zeros(1, S, N, N, dtype=torch.float32, device=s_exp.device)
    status = torch.zeros(4, dtype=torch.int32, device=s_exp.device)

    def fg(x: torch.Tensor):
        x = x.contiguous()
        status.zero_()
        if flat_samples:
            ei.ei_cost_grad_hs(plan, x[0], gamma, flat, mask, drift, s_exp, lam, cost, g[0], None, status)
        else:
            ei.ei_cost_grad_h(plan, x[0], gamma, flat, mask, drift, s_exp, lam, cost, g[0], None, status)
        return cost.clone(), g.clone()
    return fg
