"""GPU-vs-oracle parity of the paper's single-map model (NEXT-3: eq. 4, with
mu = gamma^-1 delta = h) through the C ABI: ei_forward_h and ei_cost_grad_h.  Same gates
as the three-map path (cost 1e-4 relative; s_mod, g_h and g_drift 1e-3 relative L2), on the
paper's own scan geometry P1 (220 x 220, 400 angles over 360 deg, one slope mask position,
gamma = 5, lambda = 1e-2) and a ragged case."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2202_08627_b200 import synth  # noqa: E402
import _cases  # noqa: E402


@pytest.fixture(scope="module")
def ei():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2202_08627_b200 import build
    build.build()
    from paper_2202_08627_b200 import ei as mod
    return mod


def rel_l2(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def plan_for(ei, cfg):
    return ei.Plan(cfg.S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch, cfg.z, cfg.angles)


def gpu_h(ei, plan, case, h, lam):
    cfg = case.cfg
    cost = torch.zeros(cfg.S, dtype=torch.float64, device="cuda")
    g = torch.zeros(cfg.S, cfg.N, cfg.N, device="cuda")
    gdr = torch.zeros(cfg.S, cfg.n_angles, device="cuda")
    st = torch.zeros(4, dtype=torch.int32, device="cuda")
    drift = None if case.drift is None else dev(case.drift)
    ei.ei_cost_grad_h(plan, dev(h), case.gamma, dev(case.flat), dev(case.mask), drift, dev(case.s_exp),
                      lam, cost, g, gdr, st)
    torch.cuda.synchronize()
    return cost.cpu().numpy(), g.cpu().numpy(), gdr.cpu().numpy(), st.cpu().numpy()


@pytest.mark.parametrize("name", ["P1", "RH"])
def test_forward_h_parity(ei, name):
    case = _cases.cached_h_case(name)
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    smod = torch.zeros(cfg.S, cfg.n_angles, cfg.M, cfg.n_det, device="cuda")
    drift = None if case.drift is None else dev(case.drift)
    ei.ei_forward_h(plan, dev(case.h), case.gamma, dev(case.flat), dev(case.mask), drift, smod)
    ref = _cases.ora.cost_grad_h(cfg.angles, case.h, case.gamma, case.flat, case.mask, case.drift,
                                 dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z)
    got = smod.cpu().numpy()
    for s in range(cfg.S):
        assert rel_l2(got[s], ref[s]) <= 1e-3


@pytest.mark.parametrize("name", ["P1", "RH"])
@pytest.mark.parametrize("point", ["x0", "true", "pert"])
def test_cost_grad_h_parity(ei, name, point):
    case = _cases.cached_h_case(name)
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    h = {"x0": np.zeros_like(case.h), "true": case.h,
         "pert": synth.perturbed((case.h,), cfg.seed + 7)[0]}[point]
    lam = synth.H_LAMBDA
    cost, g, gdr, st = gpu_h(ei, plan, case, h, lam)
    rc, rg, rst = _cases.oracle_cost_grad_h(case, h, lam)
    assert np.all(np.abs(cost - rc) / rc <= 1e-4), (cost, rc)
    for s in range(cfg.S):
        assert rel_l2(g[s], rg[s]) <= 1e-3, (s, rel_l2(g[s], rg[s]))
    assert st[0] == rst[0] and st[1] == rst[1]


@pytest.mark.parametrize("name", ["P1", "RH"])
def test_drift_gradient_h_parity(ei, name):
    """dS/dm_o of the single-map model: the oracle's as central differences are not exposed for
    h, so compare with the three-map oracle at (h, gamma h, 0), which has the same cost."""
    case = _cases.cached_h_case(name)
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    h = synth.perturbed((case.h,), cfg.seed + 7)[0]
    _, _, gdr, _ = gpu_h(ei, plan, case, h, 0.0)
    delta = (case.gamma * h.astype(np.float64)).astype(np.float32)
    out = _cases.ora.cost_grad(cfg.angles, h, delta, np.zeros_like(h), case.flat, case.mask, case.drift,
                               case.s_exp, 0.0, dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z, want_drift=True)
    for s in range(cfg.S):
        assert rel_l2(gdr[s], out[5][s]) <= 1e-3


def test_h_model_equals_three_map_model_on_gpu(ei):
    """The GPU's single-map path equals its three-map path at (mu, delta, sigma) = (h, gamma h, 0)
    up to the fp32 rounding of gamma h: g_h = g_mu + gamma g_delta (chain rule)."""
    case = _cases.cached_h_case("RH")
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    h = synth.perturbed((case.h,), cfg.seed + 7)[0]
    cost, g, _, _ = gpu_h(ei, plan, case, h, 0.0)
    maps = [dev(h), dev((case.gamma * h.astype(np.float64)).astype(np.float32)), dev(np.zeros_like(h))]
    drift = None if case.drift is None else dev(case.drift)
    c3, g3, _ = ei.cost_grad(plan, maps, dev(case.flat), dev(case.mask), drift, dev(case.s_exp), 0.0)
    torch.cuda.synchronize()
    assert np.all(np.abs(cost - c3.cpu().numpy()) / cost <= 1e-5)
    chain = g3[0].cpu().numpy() + case.gamma * g3[1].cpu().numpy()
    for s in range(cfg.S):
        assert rel_l2(g[s], chain[s]) <= 1e-4


@pytest.mark.parametrize("name", ["P1", "RH"])
@pytest.mark.parametrize("point", ["true", "pert"])
def test_sampled_flat_parity(ei, name, point):
    """NEXT-4: the single-map model with the measured (sampled, 33-knot) flat IC, read by a
    periodic Catmull-Rom cubic (R23): forward, cost, gradient and drift gradient vs the oracle."""
    case, fs, s_exp = _cases.cached_hs_case(name)
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    h = case.h if point == "true" else synth.perturbed((case.h,), cfg.seed + 7)[0]
    drift = None if case.drift is None else dev(case.drift)
    smod = torch.zeros(cfg.S, cfg.n_angles, cfg.M, cfg.n_det, device="cuda")
    ei.ei_forward_hs(plan, dev(h), case.gamma, dev(fs), dev(case.mask), drift, smod)
    ref = _cases.ora.cost_grad_hs(cfg.angles, h, case.gamma, fs, case.mask, case.drift,
                                  dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z)
    for s in range(cfg.S):
        assert rel_l2(smod.cpu().numpy()[s], ref[s]) <= 1e-3
    lam = synth.H_LAMBDA
    cost = torch.zeros(cfg.S, dtype=torch.float64, device="cuda")
    g = torch.zeros(cfg.S, cfg.N, cfg.N, device="cuda")
    st = torch.zeros(4, dtype=torch.int32, device="cuda")
    ei.ei_cost_grad_hs(plan, dev(h), case.gamma, dev(fs), dev(case.mask), drift, dev(s_exp), lam, cost, g,
                       None, st)
    torch.cuda.synchronize()
    rc, rg, rst = _cases.ora.cost_grad_hs(cfg.angles, h, case.gamma, fs, case.mask, case.drift, s_exp, lam,
                                          dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z)
    c = cost.cpu().numpy()
    assert np.all(np.abs(c - rc) / rc <= 1e-4), (c, rc)
    gg = g.cpu().numpy()
    for s in range(cfg.S):
        assert rel_l2(gg[s], rg[s]) <= 1e-3, (s, rel_l2(gg[s], rg[s]))
    assert list(st.cpu().numpy()[:2]) == list(rst)


def test_status_counters_h_and_sampled(ei):
    """Non-finite inputs and the P_h clamp (R12) are counted by the single-map paths exactly as
    by the oracle; the finite slice still matches."""
    case, fs, s_exp = _cases.cached_hs_case("RH")
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    h = case.h.copy()
    h[0] *= 5000.0                      # drives P_h past 50 on slice 0 (R12)
    h[1, 3, 4] = np.nan                 # one non-finite map element on slice 1
    se = s_exp.copy()
    se[1, 2, 0, 5] = np.inf
    drift = None if case.drift is None else dev(case.drift)
    cost = torch.zeros(cfg.S, dtype=torch.float64, device="cuda")
    g = torch.zeros(cfg.S, cfg.N, cfg.N, device="cuda")
    st = torch.zeros(4, dtype=torch.int32, device="cuda")
    ei.ei_cost_grad_hs(plan, dev(h), case.gamma, dev(fs), dev(case.mask), drift, dev(se), 0.0, cost, g,
                       None, st)
    torch.cuda.synchronize()
    rc, rg, rst = _cases.ora.cost_grad_hs(cfg.angles, h, case.gamma, fs, case.mask, case.drift, se, 0.0,
                                          dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z)
    assert rst[0] == 2 and rst[1] > 0
    assert list(st.cpu().numpy()[:2]) == list(rst)
    assert abs(cost.cpu().numpy()[0] - rc[0]) / rc[0] <= 1e-4
    assert rel_l2(g.cpu().numpy()[0], rg[0]) <= 1e-3


@pytest.mark.parametrize("sampled", [False, True])
def test_h_model_detector_segments(ei, sampled, monkeypatch):
    """The single-map paths (Gaussian and sampled flat) with several K2 detector segments per row
    (EI_K2_MAXW at plan creation; RH's 47 detector pixels take the lane-copy path) vs the oracle."""
    monkeypatch.setenv("EI_K2_MAXW", "16")
    case, fs, s_exp = _cases.cached_hs_case("RH")
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    assert ei.ei_plan_info(plan)["k2_segments"] > 1
    h = synth.perturbed((case.h,), cfg.seed + 7)[0]
    lam = synth.H_LAMBDA
    if sampled:
        drift = None if case.drift is None else dev(case.drift)
        cost = torch.zeros(cfg.S, dtype=torch.float64, device="cuda")
        g = torch.zeros(cfg.S, cfg.N, cfg.N, device="cuda")
        st = torch.zeros(4, dtype=torch.int32, device="cuda")
        ei.ei_cost_grad_hs(plan, dev(h), case.gamma, dev(fs), dev(case.mask), drift, dev(s_exp), lam, cost,
                           g, None, st)
        torch.cuda.synchronize()
        rc, rg, _ = _cases.ora.cost_grad_hs(cfg.angles, h, case.gamma, fs, case.mask, case.drift, s_exp, lam,
                                            dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z)
        cost, g = cost.cpu().numpy(), g.cpu().numpy()
    else:
        hc = _cases.cached_h_case("RH")
        cost, g, _, _ = gpu_h(ei, plan, hc, h, lam)
        rc, rg, _ = _cases.oracle_cost_grad_h(hc, h, lam)
    assert np.all(np.abs(cost - rc) / rc <= 1e-4), (cost, rc)
    for s in range(cfg.S):
        assert rel_l2(g[s], rg[s]) <= 1e-3, (s, rel_l2(g[s], rg[s]))


@pytest.mark.parametrize("name", ["P1", "RH"])
@pytest.mark.parametrize("band", ["0", "1"])
def test_cost_grad_h_band_and_tile_k1(ei, name, band, monkeypatch):
    """The single-map K1 in both decompositions (K1B band units, the plan's choice on P1, and the
    ray-tile units) holds the oracle gates for cost and g_h, with band heights 16 and 7 (ragged
    last band)."""
    case = _cases.cached_h_case(name)
    cfg = case.cfg
    h = synth.perturbed((case.h,), cfg.seed + 7)[0]
    lam = synth.H_LAMBDA
    rc, rg, rst = _cases.oracle_cost_grad_h(case, h, lam)
    monkeypatch.setenv("EI_K1_BAND", band)
    for br in (["16", "7"] if band == "1" else [None]):
        if br is None:
            monkeypatch.delenv("EI_K1_BR", raising=False)
        else:
            monkeypatch.setenv("EI_K1_BR", br)
        plan = plan_for(ei, cfg)
        info = ei.ei_plan_info(plan)
        assert (info["k1_band_rows"] > 0) == (band == "1")
        cost, g, gdr, st = gpu_h(ei, plan, case, h, lam)
        assert np.all(np.abs(cost - rc) / rc <= 1e-4), (br, cost, rc)
        for s in range(cfg.S):
            assert rel_l2(g[s], rg[s]) <= 1e-3, (br, s, rel_l2(g[s], rg[s]))
