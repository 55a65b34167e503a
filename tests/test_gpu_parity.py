"""GPU-vs-oracle parity through the C ABI (libei.so) — needs a B200.

Gates (BASELINE.json north_star): cost |S_gpu - S_ora| / S_ora <= 1e-4; s_mod and
each gradient map relative L2 <= 1e-3; dot test |<Rx,y> - <x,R^T y>| / max <= 1e-5 with
x, y ~ U[0,1) and fp64 inner products.  Projections alone are held to 2e-5 relative L2 (fp32
accumulation of N samples).  Evaluation points (R21): x0 = 0, x_true, x_pert.
Every input comes from paper_2202_08627_b200.synth + the fp64 oracle; nothing from the GPU.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import ora  # noqa: E402
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


def plan_for(ei, cfg, S=None):
    return ei.Plan(cfg.S if S is None else S, cfg.N, cfg.n_angles, cfg.n_det, cfg.M, cfg.pixel,
                   cfg.det_pitch, cfg.z, cfg.angles)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_cost_grad(ei, plan, case, maps, lam=0.0):
    ws = ei.Workspace(plan)
    drift = None if case.drift is None else dev(case.drift)
    cost, g, st = ei.cost_grad(plan, [dev(m) for m in maps], dev(case.flat), dev(case.mask), drift,
                               dev(case.s_exp), lam, ws)
    torch.cuda.synchronize()
    return cost.cpu().numpy(), [x.cpu().numpy() for x in g], st.cpu().numpy()


SMALL = ["C1", "C2", "R1", "R2"]


@pytest.mark.parametrize("name", SMALL)
def test_project_parity(ei, name):
    case = _cases.cached_case(name)
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    maps = np.stack(case.maps(), axis=1)                               # [S][3][N][N]
    sino = torch.zeros(cfg.S, 3, cfg.n_angles, cfg.n_det, device="cuda")
    ei.ei_project(plan, dev(maps), 3, sino)
    one = torch.zeros(cfg.S, 1, cfg.n_angles, cfg.n_det, device="cuda")
    ei.ei_project(plan, dev(maps[:, 1:2].copy()), 1, one)
    got, got1 = sino.cpu().numpy(), one.cpu().numpy()
    for s in range(cfg.S):
        for q in range(3):
            ref = ora.project(maps[s, q].astype(np.float64), cfg.angles, cfg.n_det, cfg.pixel, cfg.det_pitch)
            assert rel_l2(got[s, q], ref) < 2e-5, (s, q)
        assert np.array_equal(got1[s, 0], got[s, 1])


@pytest.mark.parametrize("name", SMALL)
def test_backproject_parity(ei, name):
    cfg = _cases.cached_case(name).cfg
    plan = plan_for(ei, cfg)
    y = synth.uniform((cfg.S, 3, cfg.n_angles, cfg.n_det), 11)
    out = torch.zeros(cfg.S, 3, cfg.N, cfg.N, device="cuda")
    ei.ei_backproject(plan, dev(y), 3, out)
    out1 = torch.zeros(cfg.S, 1, cfg.N, cfg.N, device="cuda")
    ei.ei_backproject(plan, dev(y[:, 2:3].copy()), 1, out1)
    got, got1 = out.cpu().numpy(), out1.cpu().numpy()
    for s in range(cfg.S):
        for q in range(3):
            ref = ora.backproject(y[s, q].astype(np.float64), cfg.angles, cfg.N, cfg.pixel, cfg.det_pitch)
            assert rel_l2(got[s, q], ref) < 2e-5, (s, q)
        # the single-map adjoint (pair layout) and the three-map one (triple layout, pixel pairs)
        # compute the same operator with different fp32 roundings
        assert rel_l2(got1[s, 0], got[s, 2]) < 1e-6


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5", "R1", "R2"])
def test_dot_test(ei, name):
    """<R x, y> vs <x, R^T y> with the GPU's own R and R^T (north star: <= 1e-5)."""
    cfg = synth.CONFIGS[name] if name in synth.CONFIGS else _cases.cached_case(name).cfg
    S = min(cfg.S, 2)
    plan = plan_for(ei, cfg, S)
    x = synth.uniform((S, 1, cfg.N, cfg.N), 21)
    y = synth.uniform((S, 1, cfg.n_angles, cfg.n_det), 22)
    Rx = torch.zeros(S, 1, cfg.n_angles, cfg.n_det, device="cuda")
    Rty = torch.zeros(S, 1, cfg.N, cfg.N, device="cuda")
    ei.ei_project(plan, dev(x), 1, Rx)
    ei.ei_backproject(plan, dev(y), 1, Rty)
    a = float(np.dot(Rx.cpu().numpy().astype(np.float64).ravel(), y.astype(np.float64).ravel()))
    b = float(np.dot(x.astype(np.float64).ravel(), Rty.cpu().numpy().astype(np.float64).ravel()))
    assert abs(a - b) / max(abs(a), abs(b)) <= 1e-5, (a, b)
    assert ei.ei_plan_info(plan)["window_overflows"] == 0


@pytest.mark.parametrize("name", SMALL)
def test_forward_parity(ei, name):
    case = _cases.cached_case(name)
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    smod = torch.zeros(cfg.S, cfg.n_angles, cfg.M, cfg.n_det, device="cuda")
    drift = None if case.drift is None else dev(case.drift)
    ei.ei_forward(plan, *[dev(m) for m in case.maps()], dev(case.flat), dev(case.mask), drift, smod)
    ref, _ = ora.forward(cfg.angles, *case.maps(), case.flat, case.mask, case.drift,
                         dx=cfg.pixel, du=cfg.det_pitch, z=cfg.z)
    for s in range(cfg.S):
        assert rel_l2(smod.cpu().numpy()[s], ref[s]) <= 1e-3


def eval_points(case):
    zero = tuple(np.zeros_like(m) for m in case.maps())
    return {"x0": zero, "true": case.maps(), "pert": synth.perturbed(case.maps(), case.cfg.seed + 7)}


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("point", ["x0", "true", "pert"])
def test_cost_grad_parity(ei, name, point):
    case = _cases.cached_case(name)
    plan = plan_for(ei, case.cfg)
    maps = eval_points(case)[point]
    lam = 1e-2 if point == "pert" else 0.0                              # R11: also at 1e-2
    cost, g, st = gpu_cost_grad(ei, plan, case, maps, lam)
    rc, rgm, rgd, rgs, rst = _cases.oracle_cost_grad(case, maps, lam)
    assert np.all(np.abs(cost - rc) / rc <= 1e-4), (cost, rc)
    for q, ref in enumerate((rgm, rgd, rgs)):
        for s in range(case.cfg.S):
            assert rel_l2(g[q][s], ref[s]) <= 1e-3, (q, s, rel_l2(g[q][s], ref[s]))
    assert list(st[:3]) == list(rst) and st[3] == 0
    assert ei.ei_plan_info(plan)["window_overflows"] == 0


def test_status_counters_match_oracle(ei):
    case = _cases.cached_case("R1")
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    mu, delta, sigma = (m.copy() for m in case.maps())
    mu[0] *= 4000.0                         # drives P_mu past 50 on central rays (R12)
    sigma[1] = -sigma[1] * 1e3              # negative broadening -> W^2 clamp (R13)
    delta[1, 3, 4] = np.nan                 # one non-finite map element
    s_exp = case.s_exp.copy()
    s_exp[1, 1, 0, 5] = np.inf
    c2 = synth.Case(cfg, mu, delta, sigma, case.flat, case.mask, case.drift, s_exp)
    _, _, st = gpu_cost_grad(ei, plan, c2, (mu, delta, sigma))
    _, _, _, _, rst = _cases.oracle_cost_grad(c2, (mu, delta, sigma))
    assert rst[0] == 2 and rst[1] > 0 and rst[2] > 0
    assert list(st[:3]) == list(rst)
    # the clamped but finite slice 0 still matches (the NaN only poisons slice 1)
    cost, g, _ = gpu_cost_grad(ei, plan, c2, (mu, delta, sigma))
    rc, rgm, rgd, rgs, _ = _cases.oracle_cost_grad(c2, (mu, delta, sigma), slices=[0])
    assert abs(cost[0] - rc[0]) / rc[0] <= 1e-4
    for q, ref in enumerate((rgm, rgd, rgs)):
        assert rel_l2(g[q][0], ref[0]) <= 1e-3, q


def test_launch_contract_host_path_and_determinism(ei):
    """One K1 projection and one K3 adjoint per map per evaluation;
    the host-buffer entry point equals the device one bit for bit; repeated runs are identical."""
    case = _cases.cached_case("R1")
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    s0 = ei.ei_plan_stats(plan)
    c1, g1, st1 = gpu_cost_grad(ei, plan, case, case.maps(), 1e-2)
    s1 = ei.ei_plan_stats(plan)
    info = ei.ei_plan_info(plan)   # K0, K1, K2, K3 (+ mirror fold, + angle-split reduction)
    launches = 4 + (info["mirror_pairs"] > 0) + (info["k3_angle_split"] > 1)
    assert [b - a for a, b in zip(s0, s1)] == [1, 3, 1, 3, 1, launches]
    c2, g2, _ = gpu_cost_grad(ei, plan, case, case.maps(), 1e-2)
    assert np.array_equal(c1, c2) and all(np.array_equal(a, b) for a, b in zip(g1, g2))
    S, N = cfg.S, cfg.N
    cost = np.zeros(S)
    gh = [np.zeros((S, N, N), np.float32) for _ in range(3)]
    st = np.zeros(4, np.int32)
    ei.ei_cost_grad_host(plan, *case.maps(), case.flat, case.mask, case.drift, case.s_exp, 1e-2,
                         cost, *gh, st)
    assert np.array_equal(cost, c1) and all(np.array_equal(a, b) for a, b in zip(gh, g1))
    assert np.array_equal(st, st1)


@pytest.mark.parametrize("name", ["R1", "C1", "C2"])
def test_drift_gradient_parity(ei, name):
    """NEXT-2: g_drift [S][N_theta] = dS_s/dm_o(theta) from the same pass (ei_cost_grad_drift) vs
    the oracle; the cost and map gradients are identical to ei_cost_grad's (same kernels)."""
    case = _cases.cached_case(name)
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    maps = synth.perturbed(case.maps(), cfg.seed + 7)
    drift = None if case.drift is None else dev(case.drift)
    ws = ei.Workspace(plan)
    cost, g, st, gdr = ei.cost_grad(plan, [dev(m) for m in maps], dev(case.flat), dev(case.mask),
                                    drift, dev(case.s_exp), 0.0, ws, want_drift=True)
    torch.cuda.synchronize()
    gdr = gdr.cpu().numpy().copy()
    c_d = cost.cpu().numpy().copy()
    g_d = [x.cpu().numpy().copy() for x in g]
    rc, rgm, rgd, rgs, rst, rdr = ora.cost_grad(cfg.angles, *maps, case.flat, case.mask, case.drift,
                                                case.s_exp, 0.0, dx=cfg.pixel, du=cfg.det_pitch,
                                                z=cfg.z, want_drift=True)
    for s in range(cfg.S):
        assert rel_l2(gdr[s], rdr[s]) <= 1e-3, (s, rel_l2(gdr[s], rdr[s]))
    c2, g2, _ = gpu_cost_grad(ei, plan, case, maps, 0.0)
    assert np.array_equal(c_d, c2) and all(np.array_equal(a, b) for a, b in zip(g_d, g2))


@pytest.mark.parametrize("ray_fast", ["0", "1"])
@pytest.mark.parametrize("name", ["C1", "R1"])
def test_project_parity_both_lane_mappings(ei, name, ray_fast, monkeypatch):
    """K1's two consumer lane mappings (angle fastest / ray fastest, chosen per plan by a
    bank-conflict model) give the same projections (within fp32 rounding) as the oracle."""
    monkeypatch.setenv("EI_K1_RAYFAST", ray_fast)
    case = _cases.cached_case(name)
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    info = ei.ei_plan_info(plan)
    assert info["k1_ray_fast"] == (info["k1_groups"] if ray_fast == "1" else 0)
    maps = np.stack(case.maps(), axis=1)
    sino = torch.zeros(cfg.S, 3, cfg.n_angles, cfg.n_det, device="cuda")
    ei.ei_project(plan, dev(maps), 3, sino)
    got = sino.cpu().numpy()
    for s in range(cfg.S):
        for q in range(3):
            ref = ora.project(maps[s, q].astype(np.float64), cfg.angles, cfg.n_det, cfg.pixel, cfg.det_pitch)
            assert rel_l2(got[s, q], ref) < 2e-5, (s, q)


@pytest.mark.parametrize("name", ["C2", "R1", "C5"])
def test_k1_chunking_does_not_change_projections(ei, name, monkeypatch):
    """K1 cuts each unit's rows into chunks of as many rows as fit a ring stage at the chunk's own
    window width; every ray still sums its rows one by one in row order, so the projections are
    bit-identical whatever the chunk sizes (capped at 1, 3 and 7 rows here), and match the oracle."""
    cfg = synth.CONFIGS[name] if name in synth.CONFIGS else _cases.cached_case(name).cfg
    S = min(cfg.S, 2)
    maps = synth.uniform((S, 3, cfg.N, cfg.N), 31)
    outs, rows = [], []
    for rc in (None, "1", "3", "7"):
        if rc is None:
            monkeypatch.delenv("EI_K1_RC", raising=False)
        else:
            monkeypatch.setenv("EI_K1_RC", rc)
        plan = plan_for(ei, cfg, S)
        sino = torch.zeros(S, 3, cfg.n_angles, cfg.n_det, device="cuda")
        ei.ei_project(plan, dev(maps), 3, sino)
        torch.cuda.synchronize()
        info = ei.ei_plan_info(plan)
        assert info["window_overflows"] == 0
        rows.append(info["k1_rows_per_chunk"])
        outs.append(sino.cpu().numpy())
    assert rows[1] == 1 and rows[2] <= 3 and rows[3] <= 7
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])
    ref = ora.project(maps[0, 0].astype(np.float64), cfg.angles, cfg.n_det, cfg.pixel, cfg.det_pitch)
    assert rel_l2(outs[0][0, 0], ref) < 2e-5


@pytest.mark.parametrize("name", ["C1", "C2", "R1"])
@pytest.mark.parametrize("n_maps", [3, 1])
def test_k1_angles_per_cta_do_not_change_projections(ei, name, n_maps, monkeypatch):
    """K1 CTAs of 16 angles (4 slots per thread) or 8 (2 slots, the plan's choice for grids far
    below one wave): each ray's samples are summed in the same row order either way, so the
    projections are bit-identical, for the three-map and the single-map kernels, and match the
    oracle."""
    cfg = synth.CONFIGS[name] if name in synth.CONFIGS else _cases.cached_case(name).cfg
    S = min(cfg.S, 2)
    maps = synth.uniform((S, n_maps, cfg.N, cfg.N), 37)
    outs, groups = [], []
    for nsl in ("4", "2"):
        monkeypatch.setenv("EI_K1_NSL", nsl)
        plan = plan_for(ei, cfg, S)
        sino = torch.zeros(S, n_maps, cfg.n_angles, cfg.n_det, device="cuda")
        ei.ei_project(plan, dev(maps), n_maps, sino)
        torch.cuda.synchronize()
        info = ei.ei_plan_info(plan)
        assert info["window_overflows"] == 0
        groups.append(info["k1_groups"])
        outs.append(sino.cpu().numpy())
    assert groups[1] >= 2 * groups[0] - 2          # 8-angle groups (dominance runs split both)
    assert np.array_equal(outs[0], outs[1])
    ref = ora.project(maps[0, 0].astype(np.float64), cfg.angles, cfg.n_det, cfg.pixel, cfg.det_pitch)
    assert rel_l2(outs[1][0, 0], ref) < 2e-5


@pytest.mark.parametrize("mirror", ["1", "0"])
def test_mirror_pairs_360(ei, mirror, monkeypatch):
    """360-degree scans: (theta, theta + pi) sample the same lines with the detector mirrored (R6),
    so K1 projects and K3 back-projects each pair once (gradient rows folded).  Both settings
    match the oracle (which computes every angle directly), and the dot test holds."""
    monkeypatch.setenv("EI_MIRROR", mirror)
    case = _cases.cached_case("R3")
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    assert ei.ei_plan_info(plan)["mirror_pairs"] == (20 if mirror == "1" else 0)
    maps = np.stack(case.maps(), axis=1)
    sino = torch.zeros(cfg.S, 3, cfg.n_angles, cfg.n_det, device="cuda")
    ei.ei_project(plan, dev(maps), 3, sino)
    got = sino.cpu().numpy()
    for s in range(cfg.S):
        for q in range(3):
            ref = ora.project(maps[s, q].astype(np.float64), cfg.angles, cfg.n_det, cfg.pixel, cfg.det_pitch)
            assert rel_l2(got[s, q], ref) < 2e-5, (s, q)
    y = synth.uniform((cfg.S, 3, cfg.n_angles, cfg.n_det), 12)
    out = torch.zeros(cfg.S, 3, cfg.N, cfg.N, device="cuda")
    ei.ei_backproject(plan, dev(y), 3, out)
    for s in range(cfg.S):
        for q in range(3):
            ref = ora.backproject(y[s, q].astype(np.float64), cfg.angles, cfg.N, cfg.pixel, cfg.det_pitch)
            assert rel_l2(out.cpu().numpy()[s, q], ref) < 2e-5, (s, q)
    x = synth.uniform((cfg.S, 1, cfg.N, cfg.N), 21)
    y1 = synth.uniform((cfg.S, 1, cfg.n_angles, cfg.n_det), 22)
    Rx = torch.zeros(cfg.S, 1, cfg.n_angles, cfg.n_det, device="cuda")
    Rty = torch.zeros(cfg.S, 1, cfg.N, cfg.N, device="cuda")
    ei.ei_project(plan, dev(x), 1, Rx)
    ei.ei_backproject(plan, dev(y1), 1, Rty)
    a = float(np.dot(Rx.cpu().numpy().astype(np.float64).ravel(), y1.astype(np.float64).ravel()))
    b = float(np.dot(x.astype(np.float64).ravel(), Rty.cpu().numpy().astype(np.float64).ravel()))
    assert abs(a - b) / max(abs(a), abs(b)) <= 1e-5
    mp = synth.perturbed(case.maps(), cfg.seed + 7)
    cost, g, st = gpu_cost_grad(ei, plan, case, mp, 1e-2)
    rc, rgm, rgd, rgs, rst = _cases.oracle_cost_grad(case, mp, 1e-2)
    assert np.all(np.abs(cost - rc) / rc <= 1e-4)
    for q, ref in enumerate((rgm, rgd, rgs)):
        for s in range(cfg.S):
            assert rel_l2(g[q][s], ref[s]) <= 1e-3, (q, s)


@pytest.mark.parametrize("name", ["R3", "C1"])
def test_angle_shard_partials_sum_to_full(ei, name):
    """Strong-scaling decomposition on one GPU: the per-rank plans of a 3-way
    angle shard (mirror pairs kept together), regulariser on rank 0 only, summed, equal the
    unsharded evaluation (the all-reduce itself is covered by the gloo tests)."""
    from paper_2202_08627_b200 import dist as edist
    case = _cases.cached_case(name)
    cfg = case.cfg
    maps = synth.perturbed(case.maps(), cfg.seed + 7)
    dm = [dev(m) for m in maps]
    tot_c, tot_g = 0.0, 0.0
    for r in range(3):
        sh = edist.AngleShardEval(ei, cfg, r, 3, torch.device("cuda"))
        se, dr = sh.local_inputs(case.s_exp, case.drift)
        c, g, st = sh.cost_grad(dm, dev(case.flat), dev(case.mask), dr, se, 1e-2)
        torch.cuda.synchronize()
        tot_c = tot_c + c.cpu().numpy()
        tot_g = tot_g + g.cpu().numpy()
    c_full, g_full, _ = gpu_cost_grad(ei, plan_for(ei, cfg), case, maps, 1e-2)
    assert np.all(np.abs(tot_c - c_full) / c_full <= 1e-6)
    for q in range(3):
        assert rel_l2(tot_g[q], g_full[q]) <= 1e-5


@pytest.mark.parametrize("n_det,h", [(27, False), (28, False), (27, True), (28, True)])
def test_detector_end_rows(ei, n_det, h):
    """K2's one-sided end rows of D (a2) and their transpose, where the
    rows carry signal: random maps fill the whole grid and the detector is barely wider than it
    (N_d = 27 / 28 for N = 24: corners project past both ends), unlike the ellipse phantoms whose
    sinograms vanish at the ends (R9).  N_d = 27 takes K2's lane-copy path, 28 the TMA path.
    Gates are element-wise (max |gpu - oracle| / max |oracle|), so an error confined to the
    end rows is not diluted by the L2 norm: s_mod 1e-5 (fp32 exp/rsqrt, ~1e-6 seen), gradient maps
    1e-4 (fp32 sums of N_theta * M terms), cost 1e-4 (as the north_star gate)."""
    rng = np.random.default_rng(4242 + n_det)
    S, N, NA, M = 2, 24, 13, 5
    ang = np.pi * (np.arange(NA) + 0.3) / NA
    z, w = 1.0, 0.15
    flat = np.zeros((S, 3, n_det), np.float32)
    flat[:, 0] = 1e4 * rng.uniform(0.95, 1.05, (S, n_det))
    flat[:, 1] = rng.normal(0.0, 0.05, (S, n_det))
    flat[:, 2] = w
    mask = ((np.arange(M) - (M - 1) / 2) / M).astype(np.float32)
    drift = np.cumsum(rng.normal(0.0, 0.003, NA)).astype(np.float32)
    mu = rng.uniform(0.0, 1.0, (S, N, N))
    de = rng.uniform(0.0, 1.0, (S, N, N))
    sg = rng.uniform(0.0, 1.0, (S, N, N))
    # scale as R16/R17 (oracle projector): max |z D R delta| = 0.3 w, max R sigma = (0.2 w)^2,
    # max R mu = 0.3
    for s in range(S):
        Pd = ora.project(de[s].astype(np.float32), ang, n_det)
        de[s] *= 0.3 * w / max(np.abs(z * ora.diff_t(r)).max() for r in Pd)
        sg[s] *= (0.2 * w) ** 2 / ora.project(sg[s].astype(np.float32), ang, n_det).max()
        mu[s] *= 0.3 / ora.project(mu[s].astype(np.float32), ang, n_det).max()
    if h:   # the single-map model (NEXT-3): mu = h, delta = gamma h, sigma = 0
        de, sg = synth.H_GAMMA * mu, np.zeros_like(mu)
    truth = [x.astype(np.float32) for x in (mu, de, sg)]
    s_true, _ = ora.forward(ang, *truth, flat, mask, drift, z=z)
    s_exp = (s_true * (1.0 + 0.01 * rng.standard_normal(s_true.shape))).astype(np.float32)
    maps = synth.perturbed(tuple(truth), 99)
    if h:
        maps = (maps[0], (synth.H_GAMMA * maps[0]).astype(np.float32), np.zeros_like(maps[0]))
    plan = ei.Plan(S, N, NA, n_det, M, 1.0, 1.0, z, ang)
    # forward model at the end columns
    smod = torch.zeros(S, NA, M, n_det, device="cuda")
    ei.ei_forward(plan, *[dev(m) for m in maps], dev(flat), dev(mask), dev(drift), smod)
    ref, _ = ora.forward(ang, *maps, flat, mask, drift, z=z)
    got = smod.cpu().numpy()
    ends = [0, 1, n_det - 2, n_det - 1]
    assert np.abs(got[..., ends] - ref[..., ends]).max() / np.abs(ref).max() <= 1e-5
    # cost and gradient
    rc, rgm, rgd, rgs, _ = ora.cost_grad(ang, *maps, flat, mask, drift, s_exp, 0.0, z=z)
    if h:
        cost = torch.zeros(S, dtype=torch.float64, device="cuda")
        gh = torch.zeros(S, N, N, device="cuda")
        st = torch.zeros(4, dtype=torch.int32, device="cuda")
        ei.ei_cost_grad_h(plan, dev(maps[0]), synth.H_GAMMA, dev(flat), dev(mask), dev(drift),
                          dev(s_exp), 0.0, cost, gh, None, st)
        torch.cuda.synchronize()
        pairs = [(gh.cpu().numpy(), rgm + synth.H_GAMMA * rgd)]   # dS/dh = g_mu + gamma g_delta
        cost = cost.cpu().numpy()
    else:
        ws = ei.Workspace(plan)
        cost, g, _ = ei.cost_grad(plan, [dev(m) for m in maps], dev(flat), dev(mask), dev(drift),
                                  dev(s_exp), 0.0, ws)
        torch.cuda.synchronize()
        cost = cost.cpu().numpy()
        pairs = [(x.cpu().numpy(), r) for x, r in zip(g, (rgm, rgd, rgs))]
    assert np.all(np.abs(cost - rc) / rc <= 1e-4), (cost, rc)
    for q, (a, b) in enumerate(pairs):
        err = np.abs(a - b).max() / np.abs(b).max()
        assert err <= 1e-4, (q, err)


def test_k3_angle_split_matches_unsplit(ei, monkeypatch):
    """K3's angle split (partial gradients summed in split order by ks_reduce_kernel) against one
    CTA per (tile, slice) (EI_K3_KS=1 at plan creation): the same sums in another order, so equal
    to fp32 rounding; the cost (fixed-order sums of K2's partials) is bit-identical."""
    case = _cases.cached_case("R1")
    cfg = case.cfg
    out = []
    for ks in (None, "1"):
        if ks is None:
            monkeypatch.delenv("EI_K3_KS", raising=False)
        else:
            monkeypatch.setenv("EI_K3_KS", ks)
        plan = plan_for(ei, cfg)
        out.append((ei.ei_plan_info(plan)["k3_angle_split"], gpu_cost_grad(ei, plan, case, case.maps(), 1e-2)))
    (ks_a, (ca, ga, _)), (ks_b, (cb, gb, _)) = out
    assert ks_a > 1 and ks_b == 1
    assert np.array_equal(ca, cb)
    for a, b in zip(ga, gb):
        assert rel_l2(a, b) <= 1e-6


@pytest.mark.parametrize("name,maxw", [("C1", 32), ("R1", 32), ("R1", 48), ("R3", 24)])
def test_k2_detector_segments(ei, name, maxw, monkeypatch):
    """K2 with several detector segments per row (each staged with a 4-position halo so D and D^T
    never cross segments; large configs use 2-7 segments): forced on small cases with
    EI_K2_MAXW at plan creation — C1 takes the TMA path (N_d % 4 == 0), R1 the lane-copy path,
    R3 adds mirror pairs and drift.  Same gates as test_cost_grad_parity, and the forward model."""
    monkeypatch.setenv("EI_K2_MAXW", str(maxw))
    case = _cases.cached_case(name)
    cfg = case.cfg
    plan = plan_for(ei, cfg)
    assert ei.ei_plan_info(plan)["k2_segments"] > 1
    maps = eval_points(case)["pert"]
    cost, g, st = gpu_cost_grad(ei, plan, case, maps, 1e-2)
    rc, rgm, rgd, rgs, rst = _cases.oracle_cost_grad(case, maps, 1e-2)
    assert np.all(np.abs(cost - rc) / rc <= 1e-4), (cost, rc)
    for q, ref in enumerate((rgm, rgd, rgs)):
        for s in range(cfg.S):
            assert rel_l2(g[q][s], ref[s]) <= 1e-3, (q, s, rel_l2(g[q][s], ref[s]))
    smod = torch.zeros(cfg.S, cfg.n_angles, cfg.M, cfg.n_det, device="cuda")
    drift = None if case.drift is None else dev(case.drift)
    ei.ei_forward(plan, *[dev(m) for m in maps], dev(case.flat), dev(case.mask), drift, smod)
    ref, _ = ora.forward(cfg.angles, *maps, case.flat, case.mask, case.drift, dx=cfg.pixel,
                         du=cfg.det_pitch, z=cfg.z)
    got = smod.cpu().numpy()
    assert np.abs(got - ref).max() / np.abs(ref).max() <= 1e-5


def test_project_parity_many_slices(ei):
    """K1 and K3 on a grid of several waves (128 slices: 384 K1 units, 512 K3 tiles): the work units are launched heaviest first,
    slice by slice (plan order), and every slice must still match the oracle projector / adjoint."""
    cfg = synth.small_config("RM", S=128, N=37, n_angles=29, span_deg=180.0, n_det=53, M=1, K=3, seed=61)
    plan = plan_for(ei, cfg)
    rng = np.random.default_rng(61)
    maps = rng.uniform(0.0, 1.0, (cfg.S, 3, cfg.N, cfg.N)).astype(np.float32)
    sino = torch.zeros(cfg.S, 3, cfg.n_angles, cfg.n_det, device="cuda")
    ei.ei_project(plan, dev(maps), 3, sino)
    y = rng.uniform(0.0, 1.0, (cfg.S, 3, cfg.n_angles, cfg.n_det)).astype(np.float32)
    bp = torch.zeros(cfg.S, 3, cfg.N, cfg.N, device="cuda")
    ei.ei_backproject(plan, dev(y), 3, bp)
    got, gbp = sino.cpu().numpy(), bp.cpu().numpy()
    for s in range(0, cfg.S, 7):
        for q in range(3):
            ref = ora.project(maps[s, q].astype(np.float64), cfg.angles, cfg.n_det, cfg.pixel, cfg.det_pitch)
            assert rel_l2(got[s, q], ref) < 2e-5, (s, q)
            refb = ora.backproject(y[s, q].astype(np.float64), cfg.angles, cfg.N, cfg.pixel, cfg.det_pitch)
            assert rel_l2(gbp[s, q], refb) < 2e-5, (s, q)


PLAN_MATRIX = [   # (S, N, n_angles, span_deg, n_det, M): ragged geometries that walk the plan's branches
    (1, 150, 210, 180.0, 229, 3),    # K1 single wave above the SM count -> 32-ray tiles; K3 split with extra parts
    (3, 96, 120, 360.0, 143, 2),     # mirror pairs, several slices, small K3 split
    (2, 200, 64, 180.0, 301, 5),     # sparse views: ray-fast groups
    (5, 40, 33, 360.0, 61, 1),       # odd angle count over 360 (no pairs), M = 1
    (1, 33, 17, 180.0, 50, 4),       # tiny grid: K0 triggers K1 early
]


@pytest.mark.parametrize("geom", PLAN_MATRIX)
def test_plan_matrix(ei, geom):
    """Cost and gradients vs the oracle on geometries chosen to exercise the plan's choices (ray
    tile width, row split, K3 part counts and placement, mirror pairs, lane mappings, K0's early
    launch).  Maps are random fields; s_exp is the oracle model at the maps plus 1 % noise."""
    S, N, NA, span, ND, M = geom
    cfg = synth.small_config("PM", S=S, N=N, n_angles=NA, span_deg=span, n_det=ND, M=M, K=4, seed=N + NA)
    rng = np.random.default_rng(N * 7 + NA)
    ang = cfg.angles
    mu = (rng.uniform(0.0, 1.0, (S, N, N)) * 0.3 / N).astype(np.float32)
    de = (rng.uniform(0.0, 1.0, (S, N, N)) * 0.02 / N).astype(np.float32)
    sg = (rng.uniform(0.0, 1.0, (S, N, N)) * 1e-4 / N).astype(np.float32)
    flat = np.zeros((S, 3, ND), np.float32)
    flat[:, 0] = 1e4 * rng.uniform(0.95, 1.05, (S, ND))
    flat[:, 1] = rng.normal(0.0, 0.05, (S, ND))
    flat[:, 2] = 0.15
    mask = ((np.arange(M) - (M - 1) / 2) / max(M, 1)).astype(np.float32)
    drift = np.cumsum(rng.normal(0.0, 0.002, NA)).astype(np.float32)
    s_true, _ = ora.forward(ang, mu, de, sg, flat, mask, drift)
    s_exp = (s_true * (1.0 + 0.01 * rng.standard_normal(s_true.shape))).astype(np.float32)
    maps = synth.perturbed((mu, de, sg), 5)
    plan = ei.Plan(S, N, NA, ND, M, 1.0, 1.0, 1.0, ang)
    ws = ei.Workspace(plan)
    cost, g, st = ei.cost_grad(plan, [dev(m) for m in maps], dev(flat), dev(mask), dev(drift), dev(s_exp),
                               1e-2, ws)
    torch.cuda.synchronize()
    rc, rgm, rgd, rgs, rst = ora.cost_grad(ang, *maps, flat, mask, drift, s_exp, 1e-2)
    c = cost.cpu().numpy()
    assert np.all(np.abs(c - rc) / rc <= 1e-4), (c, rc, ei.ei_plan_info(plan))
    for q, ref in enumerate((rgm, rgd, rgs)):
        gq = g[q].cpu().numpy()
        for s in range(S):
            assert rel_l2(gq[s], ref[s]) <= 1e-3, (q, s, rel_l2(gq[s], ref[s]), ei.ei_plan_info(plan))
    assert list(st.cpu().numpy()[:3]) == list(rst)


@pytest.mark.parametrize("span", [180.0, 360.0])
@pytest.mark.parametrize("chunks,n_pieces", [("3", 3), ("2", 2), ("1", 1)])
def test_host_path_chunked_stack(ei, chunks, n_pieces, span, monkeypatch):
    """Stacks: ei_cost_grad_host evaluates chunks of slices (sub-plans of the same geometry) so
    the uploads, evaluations and downloads of different chunks overlap.  Bit-identical to the
    device entry point on the same inputs (23 slices of C2's geometry in chunks of 8, 8, 7 or 12,
    11: no K3 angle split, same K1 row split), status counts equal (the shared mask/drift scanned once), one K1 launch per
    chunk; a non-finite s_exp element in slice 9 shows up in that slice's cost only.  The 360-degree
    variant (240 angles: 120 mirror pairs, folded before K3) runs the same checks."""
    monkeypatch.setenv("EI_HOST_CHUNKS", chunks)
    cfg = synth.with_slices(synth.CONFIGS["C2"], 23)
    if span == 360.0:
        import dataclasses
        cfg = dataclasses.replace(cfg, span_deg=360.0, n_angles=240)
    S, N = cfg.S, cfg.N
    rng = np.random.default_rng(5)
    sl, _ = synth.draw_slice(cfg, 0)
    maps = [np.ascontiguousarray((np.broadcast_to(m * sc, (S, N, N)) *
                                  (1 + 0.1 * rng.standard_normal((S, N, N)))).astype(np.float32))
            for m, sc in ((sl.mu, 1.0), (sl.delta, 1.0), (sl.sigma, 1.0))]
    flat = np.ascontiguousarray(np.broadcast_to(sl.flat, (S, 3, cfg.n_det))).astype(np.float32)
    mask = cfg.mask.astype(np.float32)
    drift = (0.002 * rng.standard_normal(cfg.n_angles)).astype(np.float32)
    s_exp = (rng.random((S, cfg.n_angles, cfg.M, cfg.n_det)) * 2e4).astype(np.float32)
    s_exp[9, 3, 1, 7] = np.nan
    plan = plan_for(ei, cfg)
    assert ei.ei_plan_info(plan)["mirror_pairs"] == (120 if span == 360.0 else 0)
    ws = ei.Workspace(plan)
    cost_d, g_d, st_d = ei.cost_grad(plan, [dev(m) for m in maps], dev(flat), dev(mask), dev(drift),
                                     dev(s_exp), 1e-2, ws)
    torch.cuda.synchronize()
    cost_d, g_d, st_d = cost_d.cpu().numpy(), [g.cpu().numpy() for g in g_d], st_d.cpu().numpy()

    def pinned(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    h_in = [pinned(m) for m in maps] + [pinned(flat), pinned(mask), pinned(drift), pinned(s_exp)]
    for rep in range(2):   # the first call sets up the chunks (and captures the graph), then replay
        cost = pinned(np.zeros(S))
        gh = [pinned(np.zeros((S, N, N), np.float32)) for _ in range(3)]
        st = pinned(np.zeros(4, np.int32))
        s0 = ei.ei_plan_stats(plan)
        ei.ei_cost_grad_host(plan, *h_in[:7], 1e-2, cost, *gh, st)
        s1 = ei.ei_plan_stats(plan)
        assert s1[0] - s0[0] == n_pieces, (s0, s1)
        assert np.array_equal(cost, cost_d, equal_nan=True)
        assert np.isnan(cost[9]) and np.all(np.isfinite(np.delete(cost, 9)))
        assert all(np.array_equal(a, b, equal_nan=True) for a, b in zip(gh, g_d))
        assert np.array_equal(st, st_d) and st[0] == 1


def test_host_path_many_chunks(ei, monkeypatch):
    """More than 8 chunks (the C4 default is 16): 72 slices of C2's geometry in 9 chunks of 8,
    bit-identical to the device entry point, one K1 launch per chunk, on the first call and on
    the graph replay."""
    monkeypatch.setenv("EI_HOST_CHUNKS", "9")
    cfg = synth.with_slices(synth.CONFIGS["C2"], 72)
    S, N = cfg.S, cfg.N
    rng = np.random.default_rng(8)
    maps = [(0.05 * rng.random((S, N, N))).astype(np.float32) for _ in range(3)]
    flat = np.ascontiguousarray(np.broadcast_to(synth.draw_slice(cfg, 0)[0].flat, (S, 3, cfg.n_det))).astype(np.float32)
    mask = cfg.mask.astype(np.float32)
    s_exp = (rng.random((S, cfg.n_angles, cfg.M, cfg.n_det)) * 2e4).astype(np.float32)
    plan = plan_for(ei, cfg)
    ws = ei.Workspace(plan)
    cost_d, g_d, _ = ei.cost_grad(plan, [dev(m) for m in maps], dev(flat), dev(mask), None, dev(s_exp), 1e-2, ws)
    torch.cuda.synchronize()
    cost_d, g_d = cost_d.cpu().numpy(), [g.cpu().numpy() for g in g_d]

    def pinned(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    h_in = [pinned(m) for m in maps] + [pinned(flat), pinned(mask), None, pinned(s_exp)]
    for rep in range(2):
        cost = pinned(np.zeros(S))
        gh = [pinned(np.zeros((S, N, N), np.float32)) for _ in range(3)]
        st = pinned(np.zeros(4, np.int32))
        s0 = ei.ei_plan_stats(plan)
        ei.ei_cost_grad_host(plan, *h_in[:7], 1e-2, cost, *gh, st)
        s1 = ei.ei_plan_stats(plan)
        assert s1[0] - s0[0] == 9, (s0, s1)
        assert np.array_equal(cost, cost_d)
        assert all(np.array_equal(a, b) for a, b in zip(gh, g_d))


@pytest.mark.parametrize("name", ["C1", "C2", "R1", "R3"])
def test_k1_band_mode_parity(ei, name, monkeypatch):
    """K1B band mode (units = angle group x band of BR map rows x slice; all rays swept over the
    band's fully staged rows; K2 sums the bands' partial projections in fixed order) against the
    ray-tile units and the oracle: cost, s_mod and the three gradient maps within the gates for
    band heights 5 / 16 / 1000 (ragged last band; one band = the whole map), the band and tile
    paths within fp32 rounding of each other, and repeat calls bit-identical."""
    case = _cases.cached_case(name)
    cfg = case.cfg
    maps = synth.perturbed(case.maps(), cfg.seed + 7)
    rc, rgm, rgd, rgs, rst = _cases.oracle_cost_grad(case, maps, 1e-2)
    rs, _ = ora.forward(cfg.angles, *maps, case.flat, case.mask, case.drift, dx=cfg.pixel,
                        du=cfg.det_pitch, z=cfg.z)
    runs = {}
    for band, br in (("0", None), ("1", "5"), ("1", "16"), ("1", "1000")):
        monkeypatch.setenv("EI_K1_BAND", band)
        if br is None:
            monkeypatch.delenv("EI_K1_BR", raising=False)
        else:
            monkeypatch.setenv("EI_K1_BR", br)
        plan = plan_for(ei, cfg)
        info = ei.ei_plan_info(plan)
        if band == "1":
            assert 0 < info["k1_band_rows"] <= int(br)
            assert info["k1_row_split"] == -(-cfg.N // info["k1_band_rows"])
        else:
            assert info["k1_band_rows"] == 0
        c, g, st = gpu_cost_grad(ei, plan, case, maps, 1e-2)
        c2, g2, _ = gpu_cost_grad(ei, plan, case, maps, 1e-2)
        assert np.array_equal(c, c2) and all(np.array_equal(a, b) for a, b in zip(g, g2))
        smod = torch.zeros(cfg.S, cfg.n_angles, cfg.M, cfg.n_det, device="cuda")
        drift = None if case.drift is None else dev(case.drift)
        ei.ei_forward(plan, *[dev(m) for m in maps], dev(case.flat), dev(case.mask), drift, smod)
        torch.cuda.synchronize()
        smod = smod.cpu().numpy()
        for s in range(cfg.S):
            assert abs(c[s] - rc[s]) / abs(rc[s]) <= 1e-4, (band, br, s, c[s], rc[s])
            for q, ref in enumerate((rgm, rgd, rgs)):
                assert rel_l2(g[q][s], ref[s]) <= 1e-3, (band, br, s, q, rel_l2(g[q][s], ref[s]))
        assert rel_l2(smod, rs) <= 1e-3, (band, br, rel_l2(smod, rs))
        assert list(st[:3]) == list(rst)
        runs[(band, br)] = (c, g, smod)
    c0, g0, s0 = runs[("0", None)]
    for key, (c, g, smod) in runs.items():
        assert np.allclose(c, c0, rtol=1e-6, atol=0), key
        for q in range(3):
            assert rel_l2(g[q], g0[q]) <= 1e-4, (key, q, rel_l2(g[q], g0[q]))
        assert rel_l2(smod, s0) <= 1e-5, (key, rel_l2(smod, s0))

