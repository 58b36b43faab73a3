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


class GradAllReduce:
    """The training step's one exchange: the flat fp32 gradient buffer
    (ops.AdamW packs every parameter's gradient back to back) is summed over ranks in
    fixed-size buckets issued asynchronously -- NCCL over NVLink/NVSwitch on the GPUs, so a
    bucket whose gradients are final can be reduced while the backward still runs -- and
    averaged (loss normalisation over the global batch).  `bucket_bytes` sizes buckets for
    launch latency and overlap, not for link count (NVSwitch gives every pair full bandwidth)."""

    def __init__(self, flat_grad, dist=None, bucket_bytes=32 << 20, average=True):
        self.buf = flat_grad
        self.dist = dist
        self.average = average
        n = flat_grad.numel()
        step = max(1, bucket_bytes // flat_grad.element_size())
        self.buckets = [(o, min(n, o + step)) for o in range(0, n, step)]
        self.handles = []

    def _active(self):
        return self.dist is not None and self.dist.is_initialized() and self.dist.get_world_size() > 1

    def launch(self, first=0, last=None):
        """Start the all-reduce of buckets [first, last) (their gradients are complete)."""
        if not self._active():
            return
        for o, e in self.buckets[first:last]:
            self.handles.append(self.dist.all_reduce(self.buf[o:e], op=self.dist.ReduceOp.SUM, async_op=True))

    def wait(self):
        """Wait for every launched bucket, then scale to the mean over ranks."""
        if not self._active():
            return
        for h in self.handles:
            h.wait()
        self.handles = []
        if self.average:
            self.buf.mul_(1.0 / self.dist.get_world_size())
