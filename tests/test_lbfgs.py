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
