"""Multi-process plumbing for the apply path.

Columns of X (and Mahalanobis pairs) are independent, so the path shards with no
data-path collective: each rank owns a contiguous column range (or, in the weak-scaling
bench, its own full batch).  The only collective is the max-over-ranks reduction of the
measured device time, outside the timed region.  torch.distributed is plumbing here:
`backend="nccl"` on the GPU box, `"gloo"` in the CPU tests.
"""
from __future__ import annotations

import os
from typing import Tuple

import torch
import torch.distributed as dist


def env() -> Tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 without it)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(N: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [start, stop) column range of `rank`: sizes differ by at most one and
    the ranges tile [0, N) in rank order."""
    if world < 1 or not 0 <= rank < world or N < 0:
        raise ValueError(f"bad shard request N={N} rank={rank} world={world}")
    q, r = divmod(N, world)
    start = rank * q + min(rank, r)
    return start, start + q + (1 if rank < r else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over all ranks (identity without a process group)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier() -> None:
    if dist.is_available() and dist.is_initialized():
        dist.barrier()
