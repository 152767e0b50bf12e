"""Ensemble data parallelism: one process per GPU, each rank owns
an independent slice of trajectories; there is no collective on the data path.

torch.distributed is used only for plumbing: the timing barrier and the max-over-ranks
reduction of device time (bench.py), and optional result gathering for checks.  The
functions here are host logic only, so they are exercised with the gloo backend on CPU
(tests/test_ensemble_gloo.py) as well as with NCCL on GPUs.
"""
from __future__ import annotations

import os
from typing import Optional, Tuple


def dist_env() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(rank: int, world: int, batch_per_rank: int) -> range:
    """Global element indices owned by `rank` (weak scaling: B per rank, world*B in total)."""
    if not (0 <= rank < world) or batch_per_rank < 1:
        raise ValueError("bad rank/world/batch")
    return range(rank * batch_per_rank, (rank + 1) * batch_per_rank)


def shard_of_global(rank: int, world: int, global_batch: int) -> range:
    """Contiguous split of a fixed global batch (strong scaling); remainder to the low ranks."""
    base, rem = divmod(global_batch, world)
    start = rank * base + min(rank, rem)
    return range(start, start + base + (1 if rank < rem else 0))


def init_process_group(backend: str, device=None):
    """Initialise torch.distributed from the environment if world_size > 1; returns the module or None."""
    rank, world, _ = dist_env()
    if world <= 1:
        return None
    import torch.distributed as dist
    if not dist.is_initialized():
        kw = {}
        if backend == "nccl" and device is not None:
            kw["device_id"] = device
        dist.init_process_group(backend, **kw)
    return dist


def max_over_ranks(value: float, dist, device=None) -> float:
    """Max of a per-rank scalar (device time) over all ranks; identity without a process group."""
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(world: int, cells_per_rank: int, steps: int, max_ms: float) -> float:
    """Whole-job cell-updates/s: all ranks' cells x steps over the slowest rank's device time."""
    return world * cells_per_rank * steps / (max_ms * 1e-3)


def gather_fields(local, dist, device=None) -> Optional[object]:
    """All-gather equal-shaped per-rank fields along the batch dim (checks only, off the hot path)."""
    if dist is None:
        return local
    import torch
    parts = [torch.empty_like(local) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, local)
    return torch.cat(parts, dim=0)
