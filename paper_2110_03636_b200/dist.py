"""Multi-GPU plumbing for the batch (BASELINE configs[4]):
one process per GPU, independent KKT systems sharded by rank in contiguous
blocks, torch.distributed used only for the barrier around the timed region,
the max-over-ranks of its device time and the final gather of per-system
outcomes — the systems never exchange data, so the data path has no
collective.

Sharding modes of bench.py:
  strong  a fixed global batch (256 systems = value seeds seed .. seed+255)
          split into contiguous blocks of ~global/G per rank (the north
          star's "256 systems partitioned across 1/2/4/8 GPUs");
  weak    every rank solves its own full batch of `global_batch` systems
          (disjoint seed ranges), so per-GPU work is fixed as G grows.
"""
from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(WORLD_SIZE, RANK, LOCAL_RANK) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def setup(backend: str) -> tuple[int, int, int]:
    """Initialise the process group when launched with more than one rank
    (rendezvous from MASTER_ADDR / MASTER_PORT, 127.0.0.1 on one node)."""
    w, r, lr = world()
    if w > 1:
        import torch
        import torch.distributed as dist
        if backend == "nccl":
            torch.cuda.set_device(lr)
        if not dist.is_initialized():
            dist.init_process_group(backend=backend)
    return w, r, lr


def shard_range(global_batch: int, world_size: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of the global batch owned by `rank`; the
    first global_batch % world_size ranks take one extra system."""
    base, extra = divmod(global_batch, world_size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_seeds(global_batch: int, world_size: int, rank: int, seed: int = 7,
                scaling: str = "strong") -> list[int]:
    """Value seeds of this rank's systems (system b of the job has value
    seed `seed + b`)."""
    if scaling == "strong":
        lo, hi = shard_range(global_batch, world_size, rank)
        return [seed + b for b in range(lo, hi)]
    if scaling == "weak":
        return [seed + rank * global_batch + b for b in range(global_batch)]
    raise ValueError(f"unknown scaling mode {scaling!r}")


def shard(rank: int, per_rank: int, seed: int = 7) -> list[int]:
    """Weak-scaling seeds of `rank` (disjoint across ranks)."""
    return [seed + rank * per_rank + b for b in range(per_rank)]


def _reduce(x: float, world_size: int, op: str, device=None) -> float:
    if world_size == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=getattr(dist.ReduceOp, op))
    return float(t.item())


def allmax(x: float, world_size: int, device=None) -> float:
    return _reduce(x, world_size, "MAX", device)


def allsum(x: float, world_size: int, device=None) -> float:
    return _reduce(x, world_size, "SUM", device)


def barrier(world_size: int) -> None:
    if world_size > 1:
        import torch.distributed as dist
        dist.barrier()


def gather_objects(obj, world_size: int) -> list:
    """Every rank's `obj` on every rank (per-system reports at the end)."""
    if world_size == 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * world_size
    dist.all_gather_object(out, obj)
    return out
