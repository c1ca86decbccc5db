"""Multi-GPU sweeps: replications sharded over one process per GPU.

Replications are independent (chainserve sim.py:400-404 runs them in a
process pool and merges order-independently), so each rank simulates a
contiguous block of replication indices -- each keeps its reference spawn key
(seed, rep), so results do not depend on the number of GPUs.  The only
cross-GPU traffic is the final aggregation:

* the per-replication summaries and busy times: one NCCL all-gather
  (torch.distributed on device tensors);
* the exact global quantiles: the engine's own NCCL communicator all-reduces
  the radix-select histograms and bracket counts (cs_rep_stats_dist).

Launch with torchrun (one rank per GPU), call ``init()`` once, then
``run_sim_sharded(configs)``: every rank returns the same SimStats list, equal
to ``run_sim_batch(configs)`` on one GPU.
"""

from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _native as N
from .sim import SimConfig, SimStats, _require_supported, _stats_from_batch

_initialised = False


def rank_world() -> tuple[int, int]:
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Equal contiguous replication blocks: (begin, count) of this rank."""
    if total % world:
        raise ValueError(f"replications ({total}) must be divisible by the number of GPUs ({world})")
    per = total // world
    return rank * per, per


def init() -> None:
    """Create the engine's NCCL communicator over the torch.distributed group."""
    global _initialised
    import torch
    import torch.distributed as dist

    rank, world = rank_world()
    lib = N.load()
    if world == 1:
        _initialised = True
        return
    uid = C.create_string_buffer(128)
    if rank == 0:
        N.check(lib.cs_nccl_unique_id(uid), "cs_nccl_unique_id")
    t = torch.tensor(list(uid.raw), dtype=torch.uint8, device="cuda")
    dist.broadcast(t, 0)
    raw = bytes(t.cpu().tolist())
    N.check(lib.cs_comm_init(raw, world, rank), "cs_comm_init")
    _initialised = True


def _gather_device_rows(dev, dtype, shape) -> np.ndarray:
    """Every rank's device array of `shape` ([P, R, ...], point-major) gathered
    in rank order along the replication axis: one NCCL all-gather straight
    from the device buffer and one read-back."""
    import torch
    import torch.distributed as dist

    rank, world = rank_world()
    if world == 1:
        return dev.cpu().numpy().view(dtype).reshape(shape).copy()
    flat = dev.reshape(-1)
    out = torch.empty(world * flat.numel(), dtype=flat.dtype, device=flat.device)
    dist.all_gather_into_tensor(out, flat)
    parts = out.cpu().numpy().view(dtype).reshape((world,) + tuple(shape))
    return np.concatenate(list(parts), axis=1)


def run_sim_sharded(configs: Sequence[SimConfig]) -> list[SimStats]:
    """run_sim_batch with the replications of every config split over the ranks."""
    from .engine import SweepEngine

    if not _initialised:
        init()
    c0 = configs[0]
    for c in configs:
        _require_supported(c)
        if (c.horizon_jobs, c.warmup_fraction, c.seed, c.replications) != \
                (c0.horizon_jobs, c0.warmup_fraction, c0.seed, c0.replications):
            raise ValueError("configs must share horizon, warmup, seed and replications")
        if c.collect_jobs:
            raise NotImplementedError("collect_jobs is not supported for sharded sweeps")
    rank, world = rank_world()
    begin, count = shard(c0.replications, rank, world)
    eng = SweepEngine([c.rates for c in configs], [c.capacities for c in configs],
                      [c.workload.rate for c in configs], c0.horizon_jobs, c0.warmup_fraction,
                      c0.seed, count, rep_begin=begin, distributed=world > 1,
                      total_reps=c0.replications)
    eng.step()
    return merge_sharded(configs, eng.sets[0]["summ"], eng.sets[0]["busy"], eng.order_stats(), eng.ldb)


def merge_sharded(configs: Sequence[SimConfig], local_summ, local_busy, order_stats, ldb: int) -> list[SimStats]:
    """The sharded sweep's host side: every rank's [P, R/world] summaries and
    busy times (tensors in the engine's layout) gathered in rank order along
    the replication axis, then the reference's aggregation over all
    replications (order_stats are already global: cs_rep_stats_dist)."""
    rank, world = rank_world()
    P, R = len(configs), configs[0].replications // world
    summ = _gather_device_rows(local_summ, N.SUMMARY_DTYPE, (P, R))   # [P, R_total]
    busy = _gather_device_rows(local_busy, np.float64, (P, R, ldb))
    return _stats_from_batch(configs, summ, busy, order_stats, None)
