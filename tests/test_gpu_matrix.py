"""The §8(c) parity matrix at BASELINE.json's full sizes, through the C ABI — needs a B200.

SURVEY.md §8(c) gates (BJ north_star): cost <= 1e-4 relative, s_mod and each gradient map
<= 1e-3 relative L2, on the same seeded inputs, at the evaluation points of reading R21
(x0 = 0, x_true, x_pert = x_true (1 + 0.1 U[-1,1])), on every config; for the C4 stack on every
slice.  Beside every relative-L2 gate the element-wise error max|gpu - ora| / max|ora| is
checked too (same 1e-3 bound), so an error confined to a tile edge, a K2 segment boundary or a
detector end cannot hide in the L2 norm.

* C3 and C5 (one slice each): cost and the three gradient maps at x0 (lambda = 0), x_true
  (lambda = 0, the contract's R11 value) and x_pert (lambda = 1e-2, the paper's P:93 value and
  the bench's evaluation point); s_mod (ei_forward, eq. 2/4 P:61) at x_pert.
* C4, the launch configuration bench.py times: all 64 slices drawn independently by the
  generator (seeds 4000 + s, "slice by slice"), one ei_cost_grad_drift call of the whole
  stack at x_pert with lambda = 1e-2 — cost, three gradient maps and the drift gradient
  dS_s/dm_o(theta) (NEXT-2; C4 is the only config whose flat IC drifts) of every slice,
  and their sum over the stack — and s_mod of every slice (ei_forward).
Inputs come from synth + the fp64 oracle only; nothing expected comes from the CUDA path.
"""
import dataclasses
import functools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import ora  # noqa: E402
from paper_2202_08627_b200 import synth  # noqa: E402
import _cases  # noqa: E402

TOL_COST = 1e-4
TOL = 1e-3


@pytest.fixture(scope="module")
def ei():
    assert torch.cuda.is_available()
    from paper_2202_08627_b200 import build
    build.build()
    from paper_2202_08627_b200 import ei as mod
    return mod


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def errs(a, b):
    """(relative L2, max-abs / max|ref|) of a against the reference b, in fp64."""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    d = a - b
    return (float(np.linalg.norm(d.ravel()) / max(np.linalg.norm(b.ravel()), 1e-300)),
            float(np.abs(d).max() / max(np.abs(b).max(), 1e-300)))


def gate(what, a, b, tol=TOL):
    l2, mx = errs(a, b)
    print("%-40s rel_l2 %.3e  max %.3e" % (what, l2, mx))
    assert l2 <= tol, (what, "rel_l2", l2)
    assert mx <= tol, (what, "max", mx)


def plan_for(ei, cfg):
    return ei.Plan(cfg.S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)


def eval_points(case):
    cfg = case.cfg
    zero = tuple(np.zeros_like(m) for m in case.maps())
    return {"x0": (zero, 0.0), "x_true": (case.maps(), 0.0),
            "x_pert": (synth.perturbed(case.maps(), cfg.seed + 7), 1e-2)}


@pytest.mark.parametrize("point", ["x0", "x_true", "x_pert"])
@pytest.mark.parametrize("name", ["C3", "C5"])
def test_single_slice_cost_grad(ei, name, point):
    case = _cases.cached_case(name)
    cfg = case.cfg
    maps, lam = eval_points(case)[point]
    plan = plan_for(ei, cfg)
    cost, g, st = ei.cost_grad(plan, [dev(m) for m in maps], dev(case.flat), dev(case.mask),
                               None if case.drift is None else dev(case.drift), dev(case.s_exp), lam)
    torch.cuda.synchronize()
    rc, rgm, rgd, rgs, rst = _cases.oracle_cost_grad(case, maps, lam)
    c = cost.cpu().numpy()
    rel = abs(c[0] - rc[0]) / rc[0]
    print("%s %s cost rel %.3e" % (name, point, rel))
    assert rel <= TOL_COST, (name, point, c[0], rc[0])
    for q, ref in enumerate((rgm, rgd, rgs)):
        gate("%s %s g[%d]" % (name, point, q), g[q].cpu().numpy()[0], ref[0])
    assert list(st.cpu().numpy()[:3]) == list(rst)
    assert ei.ei_plan_info(plan)["window_overflows"] == 0


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_single_slice_forward(ei, name):
    case = _cases.cached_case(name)
    cfg = case.cfg
    maps = eval_points(case)["x_pert"][0]
    plan = plan_for(ei, cfg)
    out = torch.zeros(cfg.S, cfg.n_angles, cfg.M, cfg.n_det, device="cuda")
    ei.ei_forward(plan, *[dev(m) for m in maps], dev(case.flat), dev(case.mask),
                  None if case.drift is None else dev(case.drift), out)
    torch.cuda.synchronize()
    ref, _ = ora.forward(cfg.angles, *maps, case.flat, case.mask, case.drift, dx=cfg.pixel,
                         du=cfg.det_pitch, z=cfg.z)
    gate("%s s_mod" % name, out.cpu().numpy(), ref)


@functools.lru_cache(maxsize=None)
def c4_stack():
    """The 64-slice C4 stack, every slice its own seeded phantom and flat IC (seed 4000 + s),
    the shared drift walk (seed 4999), s_exp = Poisson(oracle model) (R20)."""
    case = _cases.oracle_case(synth.CONFIGS["C4"])
    maps = synth.perturbed(case.maps(), case.cfg.seed + 7)
    return case, maps


def test_c4_stack_slices_distinct():
    case, _ = c4_stack()
    # every slice is its own problem (no repeated phantom)
    sums = {float(case.mu[s].sum()) for s in range(case.cfg.S)}
    assert len(sums) == case.cfg.S


def test_c4_stack_cost_grad_drift(ei):
    case, maps = c4_stack()
    cfg = case.cfg
    lam = 1e-2
    plan = plan_for(ei, cfg)
    cost, g, st, gdr = ei.cost_grad(plan, [dev(m) for m in maps], dev(case.flat), dev(case.mask),
                                    dev(case.drift), dev(case.s_exp), lam, want_drift=True)
    torch.cuda.synchronize()
    c = cost.cpu().numpy()
    gg = [x.cpu().numpy() for x in g]
    gd = gdr.cpu().numpy()
    assert ei.ei_plan_info(plan)["window_overflows"] == 0
    rc, rgm, rgd, rgs, rst, rdr = ora.cost_grad(cfg.angles, *maps, case.flat, case.mask, case.drift,
                                                case.s_exp, lam, dx=cfg.pixel, du=cfg.det_pitch,
                                                z=cfg.z, want_drift=True)
    worst = [0.0] * 5
    for s in range(cfg.S):
        rel = abs(c[s] - rc[s]) / rc[s]
        assert rel <= TOL_COST, (s, c[s], rc[s])
        worst[0] = max(worst[0], rel)
        for q, ref in enumerate((rgm, rgd, rgs)):
            l2, mx = errs(gg[q][s], ref[s])
            assert l2 <= TOL and mx <= TOL, (s, q, l2, mx)
            worst[1 + q] = max(worst[1 + q], l2)
        l2, mx = errs(gd[s], rdr[s])
        assert l2 <= TOL and mx <= TOL, (s, "drift", l2, mx)
        worst[4] = max(worst[4], l2)
    print("C4 x_pert worst over 64 slices: cost %.2e, g_mu %.2e, g_delta %.2e, g_sigma %.2e, "
          "g_drift %.2e" % tuple(worst))
    # the drift is shared by the stack: its gradient is the sum over slices (R25)
    gate("C4 stack drift gradient (sum over slices)", gd.astype(np.float64).sum(0), rdr.sum(0))
    assert list(st.cpu().numpy()[:3]) == list(rst)


def test_c4_stack_forward(ei):
    case, maps = c4_stack()
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    out = torch.zeros(cfg.S, cfg.n_angles, cfg.M, cfg.n_det, device="cuda")
    ei.ei_forward(plan, *[dev(m) for m in maps], dev(case.flat), dev(case.mask), dev(case.drift), out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    del out
    worst = (0.0, 0.0)
    for s0 in range(0, cfg.S, 8):                   # oracle in blocks of 8 slices (memory)
        sl = slice(s0, s0 + 8)
        sub = dataclasses.replace(cfg, S=8)
        ref, _ = ora.forward(sub.angles, *(m[sl] for m in maps), case.flat[sl], case.mask, case.drift,
                             dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z)
        for s in range(8):
            l2, mx = errs(got[s0 + s], ref[s])
            assert l2 <= TOL and mx <= TOL, (s0 + s, l2, mx)
            worst = (max(worst[0], l2), max(worst[1], mx))
    print("C4 s_mod worst over 64 slices: rel_l2 %.3e max %.3e" % worst)
