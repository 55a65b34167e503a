"""Host L-BFGS loop driving `ei_cost_grad` (the paper minimises eq. 5 with
SciPy's L-BFGS, slice by slice).  Not the hot path: every cost and
gradient comes from one C-ABI evaluation; this module only does the optimizer's vector arithmetic
(torch ops on the device) and per-problem bookkeeping (a few scalars per evaluation on the host).

Design (SPEC.md:304-305 fixes the method: two-loop recursion, history 10, strong-Wolfe line search,
stop on a relative cost decrease < 1e-9 per accepted step or max iterations; the paper gives no
optimizer parameters):
  * the unknowns are a list of BLOCKS (e.g. mu, delta, sigma, and the drift m_o for the joint
    estimation), each a tensor whose leading dimension indexes S independent PROBLEMS (the slices
    of a stack, or 1 for a stack whose slices share the drift); every problem keeps its own
    history, step length and convergence state, and all problems are evaluated together in one
    batched call;
  * two-loop recursion (history m = 10) with a block-diagonal initial matrix: one scalar
    gamma per (block, problem) from the newest pair, gamma = <s_b, y_b> / <y_b, y_b>, because the
    blocks differ by orders of magnitude and one scalar would precondition them badly (the first
    direction is the steepest-descent step of unit length per block);
  * strong-Wolfe line search per problem (Nocedal & Wright, Numerical Optimization, Alg. 3.5
    bracketing + Alg. 3.6 zoom, safeguarded cubic interpolation; c1 = 1e-4, c2 = 0.9, first
    trial step 1), so every stored pair has <s, y> > 0;
  * a problem stops when (a) its relative cost decrease over an accepted step is below rel_tol
    ("rel_tol"; a step along an L-BFGS direction that falls below it first drops the
    history, and the decision is taken on the following steepest-descent step), (b) its cost reaches `target` (a discrepancy-principle stop for
    noisy data, e.g. Morozov's S <= tau * sum s_exp for Poisson counts: "target"), (c) the line
    search finds no decrease even along steepest descent ("precision": the cost is at the
    resolution of the fp32 model), or (d) max_iter ("max_iter", converged = False).
Dot products: products in the iterate's dtype, sums in fp64.
"""
from __future__ import annotations

import dataclasses
import time
import warnings
from typing import Callable, List, Optional, Sequence, Tuple, Union

import numpy as np
import torch

Blocks = List[torch.Tensor]


@dataclasses.dataclass
class Result:
    x: Union[torch.Tensor, Blocks]  # final iterate (same structure as x0)
    cost: torch.Tensor              # [S] fp64 final cost
    history: List[torch.Tensor]     # per accepted iteration: [S] fp64 cost (history[0] = at x0)
    n_iter: int
    n_evals: int
    converged: torch.Tensor         # [S] bool
    seconds: float
    reason: List[str] = dataclasses.field(default_factory=list)   # per problem
    iters: Optional[np.ndarray] = None                             # iterations per problem


# A vector of the optimizer is either a list of block tensors [S, ...] (blocks of any shapes) or,
# when x0 is one tensor [B, S, ...] of equal blocks, that stacked tensor itself: then every vector
# operation below is one or two kernels over all blocks instead of a few per block (the loop is
# launch-bound at the sizes of one slice: ~550 launches per iteration with per-block lists).
Vec = Union[torch.Tensor, Blocks]


def _bdot(a: Vec, b: Vec) -> torch.Tensor:
    """Per-(block, problem) dot products, products in the tensors' dtype, sums in fp64: [B, S]."""
    if isinstance(a, torch.Tensor):
        return torch.sum((a * b).reshape(a.shape[0], a.shape[1], -1), dim=-1, dtype=torch.float64)
    return torch.stack([torch.sum((x * y).reshape(x.shape[0], -1), dim=-1, dtype=torch.float64)
                        for x, y in zip(a, b)])


def _sdot(a: Vec, b: Vec) -> torch.Tensor:
    """Per-problem dot products over all blocks: [S] fp64."""
    return _bdot(a, b).sum(0)


def _bc(v: torch.Tensor, like: torch.Tensor, stacked: bool = False) -> torch.Tensor:
    """Broadcast a per-problem vector [S] (or, stacked, a per-(block, problem) matrix [B, S])
    against a block [S, ...] (stacked: against the vector [B, S, ...])."""
    if v.dtype != torch.bool:
        v = v.to(like.dtype)
    if stacked and v.dim() == 1:
        return v.reshape((1,) + v.shape + (1,) * (like.dim() - 2))
    return v.reshape(v.shape + (1,) * (like.dim() - v.dim()))


def _axpy(x: Vec, a: torch.Tensor, p: Vec) -> Vec:
    """x + a p with a per-problem scalar a [S]."""
    if isinstance(x, torch.Tensor):
        return x + _bc(a, x, True) * p
    return [xb + _bc(a, xb) * pb for xb, pb in zip(x, p)]


def _where(mask: torch.Tensor, a: Vec, b: Vec) -> Vec:
    if isinstance(a, torch.Tensor):
        return torch.where(_bc(mask, a, True), a, b)
    return [torch.where(_bc(mask, xa), xa, xb) for xa, xb in zip(a, b)]


def _bscale(v: Vec, c: torch.Tensor) -> Vec:
    """v_b * c[b] with a per-(block, problem) matrix c [B, S]."""
    if isinstance(v, torch.Tensor):
        return v * _bc(c, v, True)
    return [vb * _bc(c[b], vb) for b, vb in enumerate(v)]


def _sub(a: Vec, b: Vec) -> Vec:
    return a - b if isinstance(a, torch.Tensor) else [x - y for x, y in zip(a, b)]


def _neg(a: Vec) -> Vec:
    return -a if isinstance(a, torch.Tensor) else [-x for x in a]


def _clone(a: Vec) -> Vec:
    return a.clone() if isinstance(a, torch.Tensor) else [x.clone() for x in a]


def _cubic_min(a0, f0, d0, a1, f1, d1):
    """Minimiser of the cubic interpolating (a0, f0, f'0) and (a1, f1, f'1) (N&W eq. 3.59);
    nan when it does not exist."""
    with np.errstate(all="ignore"):
        e1 = d0 + d1 - 3.0 * (f0 - f1) / (a0 - a1)
        rad = e1 * e1 - d0 * d1
        e2 = np.sign(a1 - a0) * np.sqrt(rad)
        return a1 - (a1 - a0) * (d1 + e2 - e1) / (d1 - d0 + 2.0 * e2)


def strong_wolfe(fg, x: Blocks, f0: np.ndarray, g: Blocks, p: Blocks, d0: np.ndarray,
                 active: np.ndarray, c1: float = 1e-4, c2: float = 0.9, max_ls: int = 25,
                 a_init: float = 1.0, sdot=None):
    """Batched strong-Wolfe line search (N&W Alg. 3.5 / 3.6) for every active problem along p.
    Returns (x_new, f_new [S] np, g_new, step [S] np, ok [S] bool np, n_evals): ok = a step
    satisfying sufficient decrease was found (strong Wolfe, or the best sufficient-decrease point
    when the trial budget ran out); problems not ok keep x."""
    sdot = sdot or _sdot
    S = len(f0)
    BR, ZO, DONE = 1, 2, 0
    phase = np.where(active, BR, DONE)
    a = np.full(S, a_init)
    a_prev, f_prev, d_prev = np.zeros(S), f0.copy(), d0.copy()
    a_lo, f_lo, d_lo = np.zeros(S), f0.copy(), d0.copy()
    a_hi, f_hi, d_hi = np.zeros(S), f0.copy(), d0.copy()
    best_a, best_f = np.zeros(S), f0.copy()
    found = np.zeros(S, bool)
    x_best, g_best = (x, g) if isinstance(x, torch.Tensor) else (list(x), list(g))
    n_ev = 0
    first = np.ones(S, bool)
    dev = x[0].device
    for _ in range(max_ls):
        if not (phase != DONE).any():
            break
        at = np.where(phase != DONE, a, best_a)
        at_t = torch.from_numpy(at).to(dev)
        xt = _axpy(x, at_t, p)
        ft, gt = fg(xt)
        n_ev += 1
        dt = sdot(gt, p)
        fd = torch.stack([ft.double(), dt]).cpu().numpy()
        fh, dh = fd[0], fd[1]
        upd = np.zeros(S, bool)        # this trial becomes the best sufficient-decrease point
        for s in np.nonzero(phase != DONE)[0]:
            a_s, f_s, d_s = at[s], fh[s], dh[s]
            armijo = np.isfinite(f_s) and f_s <= f0[s] + c1 * a_s * d0[s]
            wolfe = abs(d_s) <= -c2 * d0[s]
            if phase[s] == BR:
                if not armijo or (not first[s] and f_s >= f_prev[s]):
                    a_lo[s], f_lo[s], d_lo[s] = a_prev[s], f_prev[s], d_prev[s]
                    a_hi[s], f_hi[s], d_hi[s] = a_s, f_s, d_s
                    phase[s] = ZO
                elif wolfe:
                    phase[s] = DONE
                elif d_s >= 0:
                    a_lo[s], f_lo[s], d_lo[s] = a_s, f_s, d_s
                    a_hi[s], f_hi[s], d_hi[s] = a_prev[s], f_prev[s], d_prev[s]
                    phase[s] = ZO
                else:   # still descending: extrapolate (cubic, kept within [2a, 10a])
                    c = _cubic_min(a_prev[s], f_prev[s], d_prev[s], a_s, f_s, d_s)
                    a_prev[s], f_prev[s], d_prev[s] = a_s, f_s, d_s
                    a[s] = min(max(c, 2.0 * a_s), 10.0 * a_s) if np.isfinite(c) else 2.0 * a_s
                first[s] = False
            else:   # zoom
                if not armijo or f_s >= f_lo[s]:
                    a_hi[s], f_hi[s], d_hi[s] = a_s, f_s, d_s
                else:
                    if wolfe:
                        phase[s] = DONE
                    else:
                        if d_s * (a_hi[s] - a_lo[s]) >= 0:
                            a_hi[s], f_hi[s], d_hi[s] = a_lo[s], f_lo[s], d_lo[s]
                        a_lo[s], f_lo[s], d_lo[s] = a_s, f_s, d_s
            if armijo and f_s < best_f[s]:
                best_a[s], best_f[s] = a_s, f_s
                found[s] = True
                upd[s] = True
            if phase[s] == ZO:
                lo, hi = min(a_lo[s], a_hi[s]), max(a_lo[s], a_hi[s])
                c = _cubic_min(a_lo[s], f_lo[s], d_lo[s], a_hi[s], f_hi[s], d_hi[s])
                w = hi - lo
                if not np.isfinite(c) or c < lo + 0.1 * w or c > hi - 0.1 * w:
                    c = 0.5 * (lo + hi)      # safeguard: bisection
                a[s] = c
                if w <= 1e-12 * max(hi, 1e-300):   # interval collapsed: stop with the best point
                    phase[s] = DONE
        if upd.any():
            m = torch.from_numpy(upd).to(dev)
            x_best = _where(m, xt, x_best)
            g_best = _where(m, gt, g_best)
    return x_best, best_f, g_best, best_a, found, n_ev


def _as_blocks(x0) -> Tuple[Vec, bool]:
    if isinstance(x0, torch.Tensor):
        return x0, True          # stacked: the vector is the tensor [B, S, ...] itself
    return list(x0), False


def minimize(fg: Callable, x0: Union[torch.Tensor, Sequence[torch.Tensor]], max_iter: int = 200,
             m: int = 10, rel_tol: float = 1e-9, c1: float = 1e-4, c2: float = 0.9, max_ls: int = 25,
             target: Optional[Union[float, Sequence[float]]] = None,
             callback: Optional[Callable[[int, torch.Tensor, object], None]] = None,
             dot_reduce: Optional[Callable[[torch.Tensor], torch.Tensor]] = None) -> Result:
    """Minimise S independent problems.  x0: a tensor [B, S, ...] (B blocks of one shape) or a list
    of block tensors [S, ...] of any shapes; fg(x) -> (cost [S] fp64, gradient with x's structure).
    `target`: per-problem cost at which the problem stops (discrepancy principle), or None.
    `dot_reduce`: applied to every [B, S] matrix of per-block dot products — for blocks sharded over
    ranks (dist.ShardedDot) it sums their rows across ranks, so every rank takes the same steps."""
    _bdot_r = (lambda a, b: dot_reduce(_bdot(a, b))) if dot_reduce else _bdot
    _sdot_r = lambda a, b: _bdot_r(a, b).sum(0)
    t0 = time.time()
    x, stacked = _as_blocks(x0)
    x = _clone(x)
    pack = lambda v: v
    unpack = (lambda v: v) if stacked else (lambda v: list(v))
    fgb = lambda blocks: (lambda r: (r[0].double(), unpack(r[1])))(fg(pack(blocks)))
    f, g = fgb(x)
    f, g = f.clone(), _clone(g)
    n_evals = 1
    S, B = (x.shape[1], x.shape[0]) if stacked else (x[0].shape[0], len(x))
    dev = x.device if stacked else x[0].device
    Sh: List[Blocks] = []                    # history, oldest first
    Yh: List[Blocks] = []
    rho: List[torch.Tensor] = []             # [S] fp64, 0 where the pair is not valid
    gamma = torch.zeros(B, S, dtype=torch.float64, device=dev)
    has_gamma = torch.zeros(S, dtype=torch.bool, device=dev)
    fh = f.cpu().numpy().copy()
    tgt = None if target is None else np.broadcast_to(np.asarray(target, np.float64), (S,)).copy()
    done = np.zeros(S, bool)
    reason = [""] * S
    iters = np.zeros(S, int)
    if tgt is not None:
        for s in np.nonzero(fh <= tgt)[0]:
            done[s], reason[s] = True, "target"
    sd = np.ones(S, bool)                     # current direction is steepest descent
    history = [f.clone()]
    it = 0
    for it in range(1, max_iter + 1):
        if done.all():
            it -= 1
            break
        # ---- two-loop recursion: p = -H g (per problem, masked histories) ----
        q = _clone(g)
        alphas = []
        for k in reversed(range(len(Sh))):
            a_k = rho[k] * _sdot_r(Sh[k], q)
            alphas.append(a_k)
            q = _axpy(q, -a_k, Yh[k])                  # q - a_k y_k
        gnorm = _bdot_r(g, g).sqrt().clamp_min(1e-300)
        scal = torch.where(has_gamma.unsqueeze(0), gamma, 1.0 / gnorm)     # [B, S]
        r = _bscale(q, scal)
        for k, a_k in zip(range(len(Sh)), reversed(alphas)):
            b_k = rho[k] * _sdot_r(Yh[k], r)
            r = _axpy(r, a_k - b_k, Sh[k])             # r + (a_k - b_k) s_k
        p = _neg(r)
        d0 = _sdot_r(g, p)
        sd_dir = _bscale(_neg(g), scal)   # scaled steepest descent
        bad = d0 >= 0                          # not a descent direction: steepest descent
        p = _where(bad, sd_dir, p)
        d0 = torch.where(bad, _sdot_r(g, p), d0)
        db = torch.stack([d0, bad.to(d0.dtype)]).cpu().numpy()   # one device -> host transfer
        d0h, bad_h = db[0], db[1] != 0
        sd_now = sd | bad_h
        active = ~done
        x_new, f_new, g_new, step, ok, nev = strong_wolfe(fgb, x, fh, g, p, d0h, active, c1, c2, max_ls, sdot=_sdot_r)
        n_evals += nev
        # no decrease along an L-BFGS direction: retry from steepest descent next iteration (history
        # dropped); no decrease along steepest descent: converged to the model's working precision
        failed = active & ~ok
        for s in np.nonzero(failed & sd_now)[0]:
            done[s], reason[s] = True, "precision"
        # an accepted step below rel_tol along an L-BFGS direction may be a poor direction (a stale
        # or noisy curvature history) rather than convergence: drop the history and take the rel_tol
        # decision on the next, steepest-descent step
        rel = (fh - f_new) / np.maximum(np.abs(fh), 1e-300)
        acc = ok & active
        hit = acc & ((f_new <= tgt) if tgt is not None else np.zeros(S, bool))
        stall = acc & ~hit & (rel < rel_tol) & ~sd_now
        okt = torch.from_numpy(ok & active).to(dev)
        s_vec = _sub(x_new, x)
        y_vec = _sub(g_new, g)
        sy = _sdot_r(s_vec, y_vec)
        yy = _sdot_r(y_vec, y_vec)
        keep = okt & (sy > 0)
        Sh.append(s_vec)
        Yh.append(y_vec)
        rho.append(torch.where(keep, 1.0 / sy.clamp_min(1e-300), torch.zeros_like(sy)))
        if len(Sh) > m:
            Sh.pop(0), Yh.pop(0), rho.pop(0)
        reset = torch.from_numpy(failed | stall).to(dev)   # drop the history: failed or stalled
        rho = [rk * (~reset).to(rk.dtype) for rk in rho]
        gb_ = _bdot_r(s_vec, y_vec) / _bdot_r(y_vec, y_vec).clamp_min(1e-300)
        gg = (sy / yy.clamp_min(1e-300)).unsqueeze(0).expand_as(gb_)
        gb_ = torch.where(gb_ > 0, gb_, gg)             # block secant not positive: global scalar
        gamma = torch.where(keep.unsqueeze(0), gb_, gamma)
        has_gamma = has_gamma | keep    # a reset keeps the block scaling: the restart direction is
        # -gamma_b g_b, not a unit step (which overshoots badly scaled blocks by orders of magnitude)
        iters[acc] += 1
        for s in np.nonzero(acc)[0]:
            if hit[s]:
                done[s], reason[s] = True, "target"
            elif rel[s] < rel_tol and not stall[s]:
                done[s], reason[s] = True, "rel_tol"
        sd = (failed | stall) & ~done
        x, g = x_new, g_new
        fh = np.where(acc, f_new, fh)
        f = torch.from_numpy(fh.copy()).to(dev)
        history.append(f.clone())
        if callback is not None:
            callback(it, f, pack(x))
    for s in range(S):
        if not done[s]:
            reason[s] = "max_iter"
    conv = torch.from_numpy(done.copy()).to(dev)
    return Result(pack(x), f, history, it, n_evals, conv, time.time() - t0, reason, iters)


def _check_status(status: torch.Tensor, what: str):
    """a clamp is never silently active, non-finite values are an error."""
    st = status.cpu().numpy()
    if st[0]:
        raise FloatingPointError("%s: %d non-finite input elements (status[0])" % (what, int(st[0])))
    if st[1] or st[2]:
        warnings.warn("%s: clamps active (P_mu clamp %d, W^2 clamp %d; readings R12/R13)"
                      % (what, int(st[1]), int(st[2])), RuntimeWarning)


def ei_objective(plan, flat, mask, drift, s_exp, lam: float = 1e-2, ws=None, check: bool = True):
    """fg(x) for x = [3, S, N, N] (mu, delta, sigma) through the C ABI (`ei_cost_grad`).  With
    `check`, the status word is read back after every evaluation: non-finite inputs raise, active
    clamps (R12, R13) warn."""
    from . import ei
    ws = ws or ei.Workspace(plan, s_exp.device)

    def fg(x: torch.Tensor):
        x = x.contiguous()
        ws.status.zero_()
        ei.ei_cost_grad(plan, x[0], x[1], x[2], flat, mask, drift, s_exp, lam, ws.cost, ws.g[0], ws.g[1],
                        ws.g[2], ws.status)
        if check:
            _check_status(ws.status, "ei_cost_grad")
        return ws.cost.clone(), ws.g.clone()
    return fg


def ei_objective_drift(plan, flat, mask, s_exp, lam: float = 1e-2, ws=None, check: bool = True):
    """Joint estimation of the maps and the mask drift m_o(theta) of a stack (SURVEY.md §8(f)
    NEXT-2; eq. 4).  The drift is shared by the stack's slices, so the
    stack is ONE problem: x = [mu, delta, sigma, m_o] with mu/delta/sigma [1, S, N, N] and
    m_o [1, N_theta]; cost = sum over slices of S_s; dS/dm_o = sum over slices of ei_cost_grad_drift's
    per-slice drift gradient (fp64 sum; reading R25).  For a slice-sharded stack the two sums are
    the exchange across ranks (`dist.drift_allreduce`)."""
    from . import ei
    ws = ws or ei.Workspace(plan, s_exp.device)

    def fg(x: List[torch.Tensor]):
        mu, de, sg, mo = (b.contiguous() for b in x)
        ws.status.zero_()
        ei.ei_cost_grad_drift(plan, mu[0], de[0], sg[0], flat, mask, mo[0], s_exp, lam, ws.cost,
                              ws.g[0], ws.g[1], ws.g[2], ws.g_drift, ws.status)
        if check:
            _check_status(ws.status, "ei_cost_grad_drift")
        cost = ws.cost.sum().reshape(1)
        gmo = ws.g_drift.double().sum(0).float().reshape(1, -1)
        return cost, [ws.g[0].clone().unsqueeze(0), ws.g[1].clone().unsqueeze(0),
                      ws.g[2].clone().unsqueeze(0), gmo]
    return fg


def ei_objective_drift_stacked(plan, flat, mask, s_exp, lam: float = 1e-2, ws=None, check: bool = True):
    """The joint maps + drift problem of `ei_objective_drift` in the optimizer's stacked form (one
    tensor per vector, so the loop runs its one-kernel vector operations): x = [4, 1, L] with
    L = max(S N^2, N_theta); blocks 0-2 hold mu, delta, sigma flattened over the stack, block 3 the
    drift m_o(theta) in its first N_theta entries and zeros after them (their gradient is exactly 0,
    so they stay 0 and add nothing to any dot product).  Returns (fg, x0, split) with
    split(x) -> (mu, delta, sigma [S, N, N], m_o [N_theta])."""
    from . import ei
    S, N, NA, ND, M = plan.shape
    ws = ws or ei.Workspace(plan, s_exp.device)
    n, L = S * N * N, max(S * N * N, NA)
    x0 = torch.zeros(4, 1, L, device=s_exp.device)

    def split(x: torch.Tensor):
        return (x[0, 0, :n].view(S, N, N), x[1, 0, :n].view(S, N, N), x[2, 0, :n].view(S, N, N),
                x[3, 0, :NA])

    def fg(x: torch.Tensor):
        mu, de, sg, mo = split(x.contiguous())
        ws.status.zero_()
        ei.ei_cost_grad_drift(plan, mu, de, sg, flat, mask, mo, s_exp, lam, ws.cost, ws.g[0], ws.g[1],
                              ws.g[2], ws.g_drift, ws.status)
        if check:
            _check_status(ws.status, "ei_cost_grad_drift")
        g = torch.zeros_like(x0)
        g[0:3, 0, :n].copy_(ws.g.reshape(3, n))
        g[3, 0, :NA].copy_(ws.g_drift.double().sum(0).float())
        return ws.cost.sum().reshape(1), g
    return fg, x0, split


def ei_objective_h(plan, gamma: float, flat, mask, drift, s_exp, lam: float = 1e-2,
                   flat_samples: bool = False, check: bool = True):
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
        if check:
            _check_status(status, "ei_cost_grad_h")
        return cost.clone(), g.clone()
    return fg
