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


# ---------------------------------------------------------------------------------------------
# Strong scaling of ONE slice stack over its angles (single large slices such as
# C3 / C5): K1 and K2 are angle-local and K3's per-angle contributions add, so each rank evaluates
# the cost and gradient of its angles only and one all-reduce (sum) of the S x 3 x N^2 gradient
# and the S costs assembles the evaluation — the path's one real exchange step.
# ---------------------------------------------------------------------------------------------
def angle_shard(angles, rank: int, world: int):
    """Indices (ascending) of the angles rank `rank` evaluates.  Mirror pairs (theta, theta + pi
    mod 2 pi, to 1e-9 rad) stay on one rank, so its plan still projects each pair once; the
    primaries (angle mod 2 pi < pi) are split into `world` contiguous blocks in angle order,
    balanced by count, and every angle is owned by exactly one rank."""
    import numpy as np
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    a = np.asarray(angles, dtype=np.float64)
    w = np.mod(a, 2 * np.pi)
    order = np.argsort(w, kind="stable")
    partner = -np.ones(len(a), dtype=np.int64)
    used = np.zeros(len(a), dtype=bool)
    ws = w[order]
    for i in order:
        if w[i] >= np.pi or used[i]:
            continue
        lo = np.searchsorted(ws, w[i] + np.pi - 1e-9)
        for j in order[lo:]:
            if w[j] > w[i] + np.pi + 1e-9:
                break
            if j != i and not used[j]:
                partner[i] = j
                used[i] = used[j] = True
                break
    mirrors = set(int(j) for j in partner if j >= 0)
    prim = [int(i) for i in order if int(i) not in mirrors]       # primaries + unpaired, angle order
    first, count = shard(len(prim), rank, world)
    mine = []
    for i in prim[first:first + count]:
        mine.append(i)
        if partner[i] >= 0:
            mine.append(int(partner[i]))
    return np.array(sorted(mine), dtype=np.int64)


def all_reduce_sum_(*tensors) -> None:
    """In-place sum over ranks (NCCL on GPUs, gloo in tests); no-op without a process group."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return
    for t in tensors:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)


class AngleShardEval:
    """One rank's share of an angle-sharded cost + gradient evaluation through the C ABI: a plan
    over the rank's angles, its rows of s_exp and drift, the regulariser on rank 0 only, then one
    all-reduce of (gradient, cost)."""

    def __init__(self, ei, cfg, rank: int, world: int, device):
        import numpy as np
        self.ei, self.rank, self.world = ei, rank, world
        self.idx = angle_shard(cfg.angles, rank, world)
        self.plan = ei.Plan(cfg.S, cfg.N, len(self.idx), cfg.n_det, cfg.M, cfg.pixel, cfg.det_pitch,
                            cfg.z, np.ascontiguousarray(cfg.angles[self.idx]))
        self.ws = ei.Workspace(self.plan, device)
        self.device = device

    def local_inputs(self, s_exp, drift):
        """The rank's rows of s_exp [S][Na][M][Nd] and drift [Na] (numpy or torch)."""
        import numpy as np
        se = np.ascontiguousarray(np.asarray(s_exp)[:, self.idx])
        dr = None if drift is None else np.ascontiguousarray(np.asarray(drift)[self.idx])
        to = lambda a: None if a is None else torch.from_numpy(a).to(self.device)
        return to(se), to(dr)

    def cost_grad(self, maps, flat, mask, drift_local, s_exp_local, lam: float, stream=None):
        ws = self.ws
        ws.status.zero_()
        self.ei.ei_cost_grad(self.plan, maps[0], maps[1], maps[2], flat, mask, drift_local, s_exp_local,
                             lam if self.rank == 0 else 0.0, ws.cost, ws.g[0], ws.g[1], ws.g[2], ws.status,
                             stream)
        all_reduce_sum_(ws.g, ws.cost)
        return ws.cost, ws.g, ws.status


# ---------------------------------------------------------------------------------------------
# Joint drift estimation over a slice-sharded stack (R25): the
# mask drift m_o(theta) is shared by every slice of a stack, so the stack is ONE
# optimisation problem — its cost is the sum of all slices' costs and dS/dm_o the sum of all
# slices' per-slice drift gradients.  With the slices sharded over ranks these two sums are the
# exchange (N_theta + 1 fp64 values per evaluation), and the optimizer's dot products over the
# sharded map blocks are summed over ranks too, so every rank takes identical steps.
# ---------------------------------------------------------------------------------------------
def drift_allreduce(cost_local: torch.Tensor, g_drift_local: torch.Tensor):
    """(stack cost [1] fp64, stack drift gradient [N_theta] fp64) on every rank, from this rank's
    per-slice costs [S_r] and per-slice drift gradients [S_r][N_theta] (fixed-order local sums in
    fp64, then one all-reduce of N_theta + 1 values)."""
    buf = torch.cat([cost_local.double().sum().reshape(1), g_drift_local.double().sum(0)])
    all_reduce_sum_(buf)
    return buf[:1], buf[1:]


class ShardedDot:
    """dot_reduce hook for lbfgs.minimize: rows of the [B, S] per-block dot-product matrix that
    belong to blocks sharded over ranks (the maps of this rank's slices) are summed across ranks;
    replicated blocks (the drift) are already complete on every rank."""

    def __init__(self, sharded):
        self.sharded = list(bool(b) for b in sharded)

    def __call__(self, bd: torch.Tensor) -> torch.Tensor:
        if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
            return bd
        idx = [i for i, s in enumerate(self.sharded) if s]
        part = bd[idx].contiguous()
        dev = _device()
        t = part.to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        out = bd.clone()
        out[idx] = t.to(bd.device)
        return out
