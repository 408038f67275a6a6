"""Multi-GPU plumbing (one process per GPU, torch.distributed): synchronous data parallel
with mean-reduced dense gradients (§8(a) a12; S:L308-311 all_reduce_gradients) and the
per-rank batch assignment.  Collectives are NCCL on GPUs (gloo in the CPU tests); the
arithmetic of a step stays in libgsb.
"""
from __future__ import annotations

from typing import Optional

import torch


def allreduce_mean(t: torch.Tensor, group=None, world: Optional[int] = None) -> torch.Tensor:
    """In place: t <- mean over ranks of t (NCCL sum, then scale by 1/world)."""
    import torch.distributed as dist
    ws = world if world is not None else dist.get_world_size(group)
    dist.all_reduce(t, group=group)
    if ws > 1:
        t.mul_(1.0 / ws)
    return t


def rank_step(step: int, rank: int, world: int) -> int:
    """Global batch index of `step` on `rank`: rank r takes batches step*world + r, so the
    union over ranks of one step is `world` consecutive batches (a round-robin split of a
    global batch) and the RNG step word (keyed sampling) stays globally unique."""
    return step * world + rank
