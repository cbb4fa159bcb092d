"""Multi-GPU layout of the decode path.

Two partitions, neither with a data-path collective:

* ``split="sets"``: inter-frame sets are independent (keyframe-free,
  PAPER.md:158-162): set i is decoded on rank i mod world, both eyes.
* ``split="eyes"``: ranks pair up; rank 2g decodes the left eye and rank
  2g+1 the right eye of group g's frames, and sets go round-robin over the
  world/2 groups.  Both eyes come from one DWT of the top-bottom stacked
  frame (projection.py:175-179, encoding.py:395-398), so an eye's decode
  synthesises only the tiles its rows depend on -- including the other
  eye's coefficients within the lifting halo of the seam -- and its pixels
  equal the whole-frame decode's (wv_frame_args.out_row0/1).

The only exchange is the final frame gather of each rank's result (eye
images, or the decoded canvas in full-frame mode) to the display rank
(rank 0), one NCCL gather per step over NVLink.
"""
from __future__ import annotations

from dataclasses import dataclass

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


@dataclass
class Assignment:
    """One rank's share: the sets it decodes, their display frames, the eye
    it renders (None: both / mono) and the frames it completes per step."""
    sets: list
    frames: list
    eye: int | None
    frames_per_step: float


def assign(num_sets: int, inter_size: int, frame_count: int, rank: int, world: int,
           split: str = "sets", stereo: bool = True) -> Assignment:
    if split not in ("sets", "eyes"):
        raise ValueError(f"split {split!r} not in ('sets', 'eyes')")
    if split == "eyes" and stereo and world >= 2:
        if world % 2:
            raise ValueError("an eye split needs an even number of ranks")
        groups = world // 2
        sets = sets_for_rank(num_sets, rank // 2, groups)
        return Assignment(sets, frames_for_sets(sets, inter_size, frame_count), rank % 2, 0.5)
    sets = sets_for_rank(num_sets, rank, world)
    return Assignment(sets, frames_for_sets(sets, inter_size, frame_count), None, 1.0)
