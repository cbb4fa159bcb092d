"""Multi-GPU layout of the decode path.

Inter-frame sets are independent (keyframe-free): set i is
decoded on rank i mod world with no data-path collective.  The only exchange
is the final frame gather of each rank's rendered views to the display rank
(rank 0), one NCCL gather per step over NVLink.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def sets_for_rank(num_sets: int, rank: int, world: int) -> list[int]:
    """Round-robin set ownership; every rank gets at least one set."""
    own = [s for s in range(num_sets) if s % world == rank]
    return own or [rank % num_sets]


def frames_for_sets(sets: list[int], inter_size: int, frame_count: int) -> list[int]:
    """Display frames of the given sets, in order (padding frames dropped)."""
    return [s * inter_size + t for s in sets for t in range(inter_size)
            if s * inter_size + t < frame_count]


def gather_views(views: torch.Tensor, rank: int, world: int, dst: int = 0,
                 out: list | None = None) -> list | None:
    """Gather every rank's rendered views to ``dst`` (the display GPU).
    Returns the list of per-rank tensors on ``dst``, None elsewhere."""
    if world == 1:
        return [views]
    if rank == dst and out is None:
        out = [torch.empty_like(views) for _ in range(world)]
    dist.gather(views, out if rank == dst else None, dst=dst)
    return out if rank == dst else None
