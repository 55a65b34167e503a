"""Multi-process (world_size 2, gloo, CPU) tests of the slice-parallel plumbing used by bench.py
for N > 1 GPUs: sharding covers every slice once, max-over-ranks timing, cost gather order."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2202_08627_b200 import dist as edist
from paper_2202_08627_b200 import synth


def test_shard_partition():
    for n in (1, 2, 7, 64, 65):
        for world in (1, 2, 3, 8):
            owned = []
            for r in range(world):
                f, c = edist.shard(n, r, world)
                owned += list(range(f, f + c))
            assert owned == list(range(n))
    with pytest.raises(ValueError):
        edist.shard(4, 2, 2)


def test_rank_config_weak_scaling():
    cfg = synth.CONFIGS["C4"]
    assert edist.rank_config(cfg, 0) is cfg
    c1 = edist.rank_config(cfg, 1)
    assert (c1.S, c1.N, c1.n_angles) == (cfg.S, cfg.N, cfg.n_angles) and c1.seed != cfg.seed


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    edist.init("gloo")
    try:
        r, w, lr = edist.env_rank()
        assert (r, w, lr) == (rank, world, rank)
        # per-rank "device time" of a step: the slowest rank defines the step
        t = edist.max_over_ranks(1.5 + rank)
        n = 7
        first, count = edist.shard(n, rank, world)
        local = torch.arange(first, first + count, dtype=torch.float64) * 10.0 + 0.25
        full = edist.gather_costs(local, n)
        dist.barrier()
        q.put((rank, t, full.tolist()))
    finally:
        dist.destroy_process_group()


def test_world2_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for rank, t, full in res:
        assert t == 2.5
        assert full == [s * 10.0 + 0.25 for s in range(7)]


def test_angle_shard_partition_and_pairs():
    """Every angle on exactly one rank; mirror pairs (360-degree scans) kept together."""
    import numpy as np
    for cfg in (synth.CONFIGS["C3"], synth.CONFIGS["C2"], synth.small_config("R3", n_angles=40),
                synth.small_config("R1")):
        ang = cfg.angles
        for world in (1, 2, 3, 8):
            parts = [edist.angle_shard(ang, r, world) for r in range(world)]
            allidx = np.sort(np.concatenate(parts))
            assert np.array_equal(allidx, np.arange(len(ang)))
            if cfg.span_deg == 360.0 and len(ang) % 2 == 0:
                for p in parts:   # the partner theta + pi of every angle is on the same rank
                    w = np.mod(ang[p], 2 * np.pi)
                    for t in w:
                        d = np.abs(np.mod(w - t - np.pi + np.pi, 2 * np.pi) - np.pi)
                        assert d.min() < 1e-9


def _angle_worker(rank, world, port, q):
    """Each rank: the fp64 oracle's cost/gradient over its angles (regulariser on rank 0 only),
    summed over ranks with all_reduce — must equal the unsharded evaluation."""
    import numpy as np
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    edist.init("gloo")
    try:
        import _cases
        from oracle import ora
        case = _cases.cached_case("R3")
        cfg = case.cfg
        maps = synth.perturbed(case.maps(), cfg.seed + 7)
        idx = edist.angle_shard(cfg.angles, rank, world)
        lam = 1e-2 if rank == 0 else 0.0
        c, gm, gd, gs, _ = ora.cost_grad(cfg.angles[idx], *maps, case.flat, case.mask,
                                         None if case.drift is None else case.drift[idx],
                                         np.ascontiguousarray(case.s_exp[:, idx]), lam)
        cost = torch.from_numpy(c)
        g = torch.from_numpy(np.stack([gm, gd, gs]))
        edist.all_reduce_sum_(g, cost)
        q.put((rank, cost.numpy().tolist(), g.numpy()))
    finally:
        dist.destroy_process_group()


def test_angle_sharded_sum_equals_full_world2():
    import numpy as np
    import _cases
    from oracle import ora
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_angle_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    case = _cases.cached_case("R3")
    maps = synth.perturbed(case.maps(), case.cfg.seed + 7)
    rc, rgm, rgd, rgs, _ = ora.cost_grad(case.cfg.angles, *maps, case.flat, case.mask, case.drift, case.s_exp,
                                         1e-2)
    ref = np.stack([rgm, rgd, rgs])
    for rank, cost, g in res:
        np.testing.assert_allclose(cost, rc, rtol=1e-12)
        assert np.linalg.norm(g - ref) / np.linalg.norm(ref) < 1e-12


def _drift_worker(rank, world, port, q, iters):
    """Joint map + drift estimation of one stack sharded by slices (rank r owns slice r): the
    oracle's cost and drift gradient of the rank's slice, summed over ranks (dist.drift_allreduce),
    and the optimizer's dot products over the sharded map blocks summed too (dist.ShardedDot)."""
    import numpy as np
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    edist.init("gloo")
    try:
        import _cases
        from paper_2202_08627_b200 import lbfgs
        import test_recon_oracle as tro
        case = tro.drift_case(noise=False)
        cfg = case.cfg
        first, count = edist.shard(cfg.S, rank, world)
        local = _cases.oracle_objective_drift(case, 0.0, slices=range(first, first + count))

        def fg(x):
            c, g = local(x)
            ct, gdr = edist.drift_allreduce(c, g[3])
            return ct, g[:3] + [gdr.reshape(1, -1)]
        x0 = ([torch.zeros(1, count, cfg.N, cfg.N, dtype=torch.float64) for _ in range(3)] +
              [torch.zeros(1, cfg.n_angles, dtype=torch.float64)])
        res = lbfgs.minimize(fg, x0, max_iter=iters, dot_reduce=edist.ShardedDot([1, 1, 1, 0]))
        q.put((rank, float(res.cost[0]), res.x[3][0].numpy(), res.x[0][0].numpy(), res.n_iter))
    finally:
        dist.destroy_process_group()


def test_sharded_joint_drift_world2():
    import numpy as np
    import _cases
    from paper_2202_08627_b200 import lbfgs
    import test_recon_oracle as tro
    iters = 25
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_drift_worker, args=(r, world, port, q, iters)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    case = tro.drift_case(noise=False)
    ref = lbfgs.minimize(_cases.oracle_objective_drift(case, 0.0), tro.drift_x0(case.cfg), max_iter=iters)
    # every rank took the same steps: identical drift and stack cost on both ranks
    assert res[0][1] == res[1][1] and np.array_equal(res[0][2], res[1][2])
    # and the same steps as the unsharded optimisation (up to the order of the fp64 sums)
    assert abs(res[0][1] - float(ref.cost[0])) <= 1e-6 * float(ref.cost[0])
    mo = ref.x[3][0].numpy()
    assert np.linalg.norm(res[0][2] - mo) <= 1e-4 * np.linalg.norm(mo)
    maps = np.concatenate([res[0][3], res[1][3]])
    assert np.linalg.norm(maps - ref.x[0][0].numpy()) <= 1e-4 * np.linalg.norm(maps)
