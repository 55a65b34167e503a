"""The plan's size limits, and parity at them (include/ei.h: 16 N_d + 4 M <= 225280, N_theta <=
14080; K2's staging ring bounds M).  Each limit is exercised where it is the only large dimension, so the
fp64 oracle still finishes in seconds:
* N_d = 14079 at M = 3 (K2 in many detector segments, K1/K3 windows at the detector's far ends);
* N_theta = 14080 (K1 angle groups, K3 angle chunks, the per-angle drift gradient);
* the largest M the plan accepts for a small geometry (K2's per-item rows);
and the first size past each limit is refused with EI_ERR_SHAPE before any launch."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import ora  # noqa: E402

NA_MAX = 14080


def nd_max(M):
    return (220 * 1024 - 4 * M) // 16


@pytest.fixture(scope="module")
def ei():
    assert torch.cuda.is_available()
    from paper_2202_08627_b200 import build
    build.build()
    from paper_2202_08627_b200 import ei as mod
    return mod


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def plan_or_code(ei, S, N, ang, ND, M):
    try:
        return ei.Plan(S, N, len(ang), ND, M, 1.0, 1.0, 1.0, ang), 0
    except ei.EIError as e:
        return None, e.code


def check_parity(ei, S, N, ang, ND, M, seed):
    rng = np.random.default_rng(seed)
    maps = [rng.uniform(0, 0.05, (S, N, N)).astype(np.float32),
            rng.uniform(0, 0.02, (S, N, N)).astype(np.float32),
            rng.uniform(0, 3e-4, (S, N, N)).astype(np.float32)]
    flat = np.stack([1e4 * (1 + rng.uniform(-0.05, 0.05, (S, ND))), rng.normal(0, 0.05, (S, ND)),
                     np.full((S, ND), 0.15)], axis=1).astype(np.float32)
    mask = ((np.arange(M) - (M - 1) / 2) / M).astype(np.float32)
    drift = rng.normal(0, 0.01, len(ang)).astype(np.float32)
    s_exp = rng.uniform(0, 1.1e4, (S, len(ang), M, ND)).astype(np.float32)
    plan, code = plan_or_code(ei, S, N, ang, ND, M)
    assert code == 0
    ws = ei.Workspace(plan)
    cost, g, st, gdr = ei.cost_grad(plan, [dev(m) for m in maps], dev(flat), dev(mask), dev(drift),
                                    dev(s_exp), 1e-2, ws, want_drift=True)
    torch.cuda.synchronize()
    rc, rgm, rgd, rgs, rst, rdr = ora.cost_grad(ang, *maps, flat, mask, drift, s_exp, 1e-2, want_drift=True)
    c = cost.cpu().numpy()
    for s in range(S):
        assert abs(c[s] - rc[s]) / rc[s] <= 1e-4, (s, c[s], rc[s])
        for q, ref in enumerate((rgm, rgd, rgs)):
            got = g[q].cpu().numpy()[s]
            assert rel_l2(got, ref[s]) <= 1e-3, (s, q)
            assert np.abs(got - ref[s]).max() <= 1e-3 * np.abs(ref[s]).max(), (s, q)
    assert rel_l2(gdr.cpu().numpy(), rdr) <= 1e-3
    assert np.array_equal(st.cpu().numpy()[:3], np.asarray(rst)[:3])
    assert ei.ei_plan_info(plan)["window_overflows"] == 0
    # projector and adjoint alone, against the oracle
    x = rng.uniform(0, 1, (S, 1, N, N)).astype(np.float32)
    y = rng.uniform(0, 1, (S, 1, len(ang), ND)).astype(np.float32)
    Rx = torch.zeros(S, 1, len(ang), ND, device="cuda")
    Rty = torch.zeros(S, 1, N, N, device="cuda")
    ei.ei_project(plan, dev(x), 1, Rx)
    ei.ei_backproject(plan, dev(y), 1, Rty)
    torch.cuda.synchronize()
    assert rel_l2(Rx.cpu().numpy()[0, 0], ora.project(x[0, 0].astype(np.float64), ang, ND, 1.0, 1.0)) < 2e-5
    assert rel_l2(Rty.cpu().numpy()[0, 0], ora.backproject(y[0, 0].astype(np.float64), ang, N, 1.0, 1.0)) < 2e-5
    return plan


def test_limits_refused_past_the_boundary(ei):
    ang = np.linspace(0, np.pi, 8, endpoint=False)
    for M in (1, 3, 7):
        assert plan_or_code(ei, 1, 16, ang, nd_max(M), M)[1] == 0
        assert plan_or_code(ei, 1, 16, ang, nd_max(M) + 1, M)[1] == 2
    many = np.linspace(0, np.pi, NA_MAX, endpoint=False)
    assert plan_or_code(ei, 1, 16, many, 24, 2)[1] == 0
    assert plan_or_code(ei, 1, 16, np.linspace(0, np.pi, NA_MAX + 1, endpoint=False), 24, 2)[1] == 2


def test_parity_at_max_detector(ei):
    """N_d = 14079 (M = 3) on a 96 x 96 slice: most rays miss the map (zero projections, flat curves),
    the K2 rows run in many segments and every detector end row is exercised."""
    ang = np.deg2rad(np.array([0.0, 10.0, 33.0, 45.0, 71.0, 90.0, 118.0, 135.0, 160.0, 179.0]))
    assert nd_max(3) == 14079
    plan = check_parity(ei, 1, 96, ang, nd_max(3), 3, 101)
    assert ei.ei_plan_info(plan)["k2_segments"] > 1


def test_parity_at_max_angles(ei):
    """N_theta = 14080 angles (irregular, over 360 degrees, two slices) on a 16 x 16 slice."""
    rng = np.random.default_rng(7)
    ang = np.sort(rng.uniform(0, 2 * np.pi, NA_MAX))
    check_parity(ei, 2, 16, ang, 24, 2, 102)


def test_parity_at_max_mask_positions(ei):
    """The largest M the plan accepts for a 32 x 32 slice with 64 detector pixels (found by
    bisection on plan creation), then parity there; M + 1 is refused with EI_ERR_SHAPE."""
    ang = np.linspace(0, np.pi, 12, endpoint=False)
    lo, hi = 1, 1 << 14
    assert plan_or_code(ei, 1, 32, ang, 64, lo)[1] == 0
    assert plan_or_code(ei, 1, 32, ang, 64, hi)[1] == 2
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if plan_or_code(ei, 1, 32, ang, 64, mid)[1] == 0:
            lo = mid
        else:
            hi = mid
    assert lo >= 33                                 # at least the paper's 33 mask steps
    check_parity(ei, 1, 32, ang, 64, lo, 103)
