"""CPU tests of the host L-BFGS loop (paper_2202_08627_b200/lbfgs.py) on analytic problems:
independent quadratics with badly scaled blocks (the regime of mu/delta/sigma) and a Rosenbrock
valley, several slices at once with different conditioning."""
import torch

from paper_2202_08627_b200 import lbfgs


def quad_problem(S=3, B=3, n=40, seed=0):
    g = torch.Generator().manual_seed(seed)
    scales = torch.tensor([1.0, 1e-2, 1e-4], dtype=torch.float64)[:B]
    # per (block, slice) diagonal Hessians with condition ~100 inside a block
    H = (torch.rand(B, S, n, generator=g, dtype=torch.float64) * 99 + 1) / scales.view(B, 1, 1) ** 2
    xs = torch.randn(B, S, n, generator=g, dtype=torch.float64) * scales.view(B, 1, 1)

    def fg(x):
        d = x.double() - xs
        f = 0.5 * (H * d * d).sum(dim=(0, 2))
        return f, (H * d).to(x.dtype)
    return fg, xs


def test_quadratic_blocks_converge():
    fg, xs = quad_problem()
    x0 = torch.zeros_like(xs)
    res = lbfgs.minimize(fg, x0, max_iter=300, rel_tol=1e-14)
    f0, _ = fg(x0)
    assert torch.all(res.cost <= 1e-10 * f0)
    for b in range(3):
        err = (res.x[b] - xs[b]).norm() / xs[b].norm()
        assert err < 1e-4, (b, float(err))
    # monotone: every accepted step decreases every slice's cost (Armijo)
    for a, b in zip(res.history, res.history[1:]):
        assert torch.all(b <= a)


def test_rosenbrock_slices():
    S = 4
    shift = torch.linspace(0.5, 2.0, S, dtype=torch.float64)

    def fg(x):   # x: [2, S, 1]; minimum at (shift, shift^2)
        a, b = x[0, :, 0], x[1, :, 0]
        f = (shift - a) ** 2 + 100 * (b - a * a) ** 2
        ga = -2 * (shift - a) - 400 * a * (b - a * a)
        gb = 200 * (b - a * a)
        return f, torch.stack([ga, gb]).unsqueeze(-1)
    x0 = torch.zeros(2, S, 1, dtype=torch.float64)
    res = lbfgs.minimize(fg, x0, max_iter=500, rel_tol=1e-16)
    assert torch.all(res.cost < 1e-10), res.cost
    assert torch.allclose(res.x[0, :, 0], shift, atol=1e-4)
    assert res.n_iter < 500


# ---------------------------------------------------------------------------------------------
# strong-Wolfe line search, mixed-shape blocks, stopping rules
# ---------------------------------------------------------------------------------------------
def test_strong_wolfe_conditions_hold():
    """Every accepted step of the batched line search satisfies both strong-Wolfe conditions
    (N&W eq. 3.7): phi(a) <= phi(0) + c1 a phi'(0) and |phi'(a)| <= c2 |phi'(0)|, on problems
    needing extrapolation (minimiser far beyond a = 1), interpolation (minimiser well inside)
    and a non-quadratic valley."""
    import numpy as np
    c1, c2 = 1e-4, 0.9
    targets = torch.tensor([30.0, 0.05, 1.0, -3.0], dtype=torch.float64)   # per problem

    def fg(xb):
        x = xb[0]
        d = x - targets.view(-1, 1)
        f = (d ** 2).sum(1) + 0.1 * (d ** 4).sum(1)
        return f, [2 * d + 0.4 * d ** 3]
    x = [torch.zeros(4, 1, dtype=torch.float64)]
    f0, g0 = fg(x)
    p = [torch.sign(targets).view(-1, 1)]                       # unit descent directions
    d0 = (g0[0] * p[0]).sum(1)
    assert torch.all(d0 < 0)
    xn, fn, gn, step, ok, nev = lbfgs.strong_wolfe(fg, x, f0.numpy(), g0, p, d0.numpy(),
                                                    np.ones(4, bool), c1, c2)
    assert ok.all()
    dn = (gn[0] * p[0]).sum(1).numpy()
    for s in range(4):
        assert fn[s] <= f0[s].item() + c1 * step[s] * d0[s].item() + 1e-12
        assert abs(dn[s]) <= c2 * abs(d0[s].item()) + 1e-12, (s, step[s], dn[s], d0[s])
    assert step[0] > 1.0 and step[1] < 1.0                      # extrapolated / interpolated
    assert torch.allclose(xn[0], x[0] + torch.from_numpy(step).view(-1, 1) * p[0])


def test_mixed_blocks_list_form():
    """Blocks of different shapes (maps [S, n, n] and a per-problem vector [S, k], like the maps
    and the drift of the joint estimation) in the list form, two problems at once."""
    g = torch.Generator().manual_seed(3)
    S = 2
    A = torch.rand(S, 5, 5, generator=g, dtype=torch.float64) + 0.5
    xa = torch.randn(S, 5, 5, generator=g, dtype=torch.float64) * 1e-3
    xb = torch.randn(S, 7, generator=g, dtype=torch.float64) * 10.0

    def fg(x):
        da, db = x[0] - xa, x[1] - xb
        f = (A * da * da).sum((1, 2)) * 1e6 + 0.5 * (db * db).sum(1) + 1e-3 * (da.sum((1, 2)) * db.sum(1))
        ga = 2e6 * A * da + 1e-3 * db.sum(1).view(S, 1, 1)
        gb = db + 1e-3 * da.sum((1, 2)).view(S, 1)
        return f, [ga, gb]
    res = lbfgs.minimize(fg, [torch.zeros_like(xa), torch.zeros_like(xb)], max_iter=500, rel_tol=1e-15)
    assert isinstance(res.x, list) and res.x[0].shape == xa.shape and res.x[1].shape == xb.shape
    assert (res.x[0] - xa).norm() / xa.norm() < 1e-4
    assert (res.x[1] - xb).norm() / xb.norm() < 1e-4
    for a, b in zip(res.history, res.history[1:]):
        assert torch.all(b <= a)


def test_target_stop_and_reasons():
    """The discrepancy-principle stop: a problem stops at the first accepted iterate whose cost is
    <= its target (reason "target"); the other problem runs on to rel_tol."""
    fg, xs = quad_problem(S=2)
    x0 = torch.zeros_like(xs)
    f0 = fg(x0)[0]
    res = lbfgs.minimize(fg, x0, max_iter=500, rel_tol=1e-12, target=[1e-3 * float(f0[0]), 0.0])
    assert res.reason[0] == "target" and float(res.cost[0]) <= 1e-3 * float(f0[0])
    assert float(res.history[res.iters[0] - 1][0]) > 1e-3 * float(f0[0])   # the first one below
    assert res.reason[1] in ("rel_tol", "precision") and bool(res.converged.all())
    assert res.iters[1] > res.iters[0]


def test_stacked_and_list_forms_take_the_same_steps():
    """The same problem given as one stacked tensor [B, S, n] (the fast path: one kernel per
    vector operation over all blocks) and as a list of B block tensors takes the same iterates:
    the two paths differ only in how the fp64 per-block sums are blocked, so the costs agree to
    rounding along the whole run and both converge to the minimiser."""
    fg, xs = quad_problem(S=2, B=3, n=30, seed=5)
    x0 = torch.zeros_like(xs)
    rs = lbfgs.minimize(fg, x0, max_iter=60, rel_tol=0.0)

    def fg_list(blocks):
        f, g = fg(torch.stack(blocks))
        return f, [g[b] for b in range(g.shape[0])]
    rl = lbfgs.minimize(fg_list, [x0[b].clone() for b in range(x0.shape[0])], max_iter=60, rel_tol=0.0)
    assert isinstance(rs.x, torch.Tensor) and isinstance(rl.x, list)
    assert rs.n_iter == rl.n_iter and rs.n_evals == rl.n_evals
    for a, b in zip(rs.history, rl.history):
        assert torch.allclose(a, b, rtol=1e-9, atol=0.0)
    for b in range(3):
        assert torch.allclose(rs.x[b], rl.x[b], rtol=1e-7, atol=1e-12 * float(xs[b].abs().max()))
