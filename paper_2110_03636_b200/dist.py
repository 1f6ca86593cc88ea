"""Multi-GPU plumbing for the batch (BASELINE configs[4]): one process per
GPU, independent systems sharded by rank, torch.distributed used only for
the barrier and the max-over-ranks of the timed region — the systems never
exchange data, so there is no collective on the data path."""
from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(rank: int, per_rank: int, seed: int = 7) -> list[int]:
    """Value seeds of this rank's systems: disjoint across ranks."""
    return [seed + rank * per_rank + b for b in range(per_rank)]


def allmax(x: float, world_size: int, device=None) -> float:
    if world_size == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allsum(x: float, world_size: int, device=None) -> float:
    if world_size == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
