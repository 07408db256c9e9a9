"""Host-side plumbing for N > 1 ranks (one process per GPU, torch.distributed).

The collision step shards by cells with no data-path collective (cells are independent): each rank
owns a disjoint cell range (strong split of one batch) or its own box (weak scaling, what bench.py does).
The only collective is the max-over-ranks of the device-measured step time.
"""
from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 without it)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n: int, rank: int, size: int) -> tuple[int, int]:
    """Contiguous, disjoint, balanced cell range [a, b) of rank `rank` among `size` ranks (covers [0, n))."""
    if size < 1 or not 0 <= rank < size:
        raise ValueError("bad rank/size")
    base, extra = divmod(n, size)
    a = rank * base + min(rank, extra)
    return a, a + base + (1 if rank < extra else 0)


def rank_seed(rank: int) -> int | None:
    """Input seed of a rank's own box under weak scaling (rank 0 reproduces the single-GPU workload)."""
    return None if rank == 0 else rank


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank scalar (device-timed milliseconds) over all ranks; identity without a process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def weak_value(cells_per_rank: int, n_velocity: int, size: int, ms_max: float, steps: int = 1) -> float:
    """Whole-job throughput: cells·velocity-points processed by ALL ranks / slowest rank's time."""
    return cells_per_rank * n_velocity * size * steps / (ms_max / 1e3)
