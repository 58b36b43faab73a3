"""Multi-GPU plumbing for the hot path.

Every hot-path op is per image (index, attention and merge never mix images), so
the batch shards by image with NO data-path collective: rank g owns global images
[g*B, (g+1)*B) and derives every seed from the global image index, so results do
not depend on the number of ranks.  The only collectives are timing reductions
(max over ranks) and, in a training step, the gradient all-reduce.
"""
from __future__ import annotations


def image_range(images_per_rank: int, rank: int, world: int) -> range:
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world {world}")
    return range(rank * images_per_rank, (rank + 1) * images_per_rank)


def mask_seed(global_image: int, seed0: int = 1000) -> int:
    """Perlin-mask seed of a global image (Rng(1000 + b))."""
    return seed0 + global_image


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (device time) over all ranks; identity without dist."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None, device=None) -> float:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
