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
