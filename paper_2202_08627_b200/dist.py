"""Multi-GPU plumbing for slice-parallel evaluation (torch.distributed; NCCL on GPUs, gloo in tests).

Slices are independent reconstruction problems ("works independently on each
220x220 slice"), so the cost+gradient path shards with NO collective on the data path:
  * weak scaling (bench.py): every rank evaluates its own seeded slice stack (`rank_config`);
  * strong scaling of one stack: `shard(S, rank, world)` gives each rank a contiguous block of
    slices; per-slice costs are assembled with `gather_costs` (host metadata only).
The only collectives are host-side: the timing barrier, `max_over_ranks` for the device time of
a step (the slowest rank defines the step) and the optional cost gather.
"""
from __future__ import annotations

import dataclasses
import os
from typing import Tuple

import torch
import torch.distributed as dist


def env_rank() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str, device=None) -> None:
    """Initialise the default process group from the environment (MASTER_ADDR/PORT set by torchrun)."""
    if dist.is_initialized():
        return
    kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
    dist.init_process_group(backend, **kw)


def shard(n_slices: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block partition of n_slices over world ranks: (first, count); the first
    n_slices % world ranks get one extra slice.  Every slice is owned by exactly one rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_slices, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def rank_config(cfg, rank: int):
    """Weak scaling: rank r evaluates its own stack, seeded cfg.seed + 100000 r (same shapes)."""
    return cfg if rank == 0 else dataclasses.replace(cfg, seed=cfg.seed + 100000 * rank)


def _device():
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")


def max_over_ranks(x: float) -> float:
    """Max of a host scalar over all ranks (identity without a process group)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_costs(local_costs: torch.Tensor, n_slices: int) -> torch.Tensor:
    """Assemble per-slice fp64 costs of a sharded stack (each rank holds its `shard`) in slice
    order on every rank."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local_costs.to(torch.float64).cpu()
    world, rank = dist.get_world_size(), dist.get_rank()
    dev = _device()
    full = torch.zeros(n_slices, dtype=torch.float64, device=dev)
    first, count = shard(n_slices, rank, world)
    full[first:first + count] = local_costs.to(device=dev, dtype=torch.float64)
    dist.all_reduce(full, op=dist.ReduceOp.SUM)   # disjoint supports: a gather, exact in fp64
    return full.cpu()
