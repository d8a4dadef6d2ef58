"""Multi-GPU plumbing for the frame-parallel path.

Frames are independent codewords of one shared code, so N GPUs decode N
disjoint frame ranges with no collective on the data path (weak scaling: each
rank keeps its own batch).  The only collectives are host-side bookkeeping:
the max-over-ranks timing and optional gathers of per-frame results.
"""
from __future__ import annotations


def frame_range(rank: int, world: int, frames_per_rank: int) -> range:
    """Frame ids of `rank` in the config's seeded stream: [rank*F, (rank+1)*F)."""
    if not (0 <= rank < world) or frames_per_rank < 0:
        raise ValueError("bad rank / world / frame count")
    return range(rank * frames_per_rank, (rank + 1) * frames_per_rank)


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (timings are reported as the slowest rank)."""
    if dist is None or not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    if dist is None or not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_objects(obj, dist=None):
    """All ranks' `obj` in rank order (a list of length world)."""
    if dist is None or not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out
