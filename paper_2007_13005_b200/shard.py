"""Per-GPU sharding of an image batch.

Images are independent units: the batch is partitioned into contiguous
ranges, one per rank, balanced by ROI block count (the decode work of an
image under the plan), and every rank runs the fused kernel on its own range.
There is no data-path collective and no NCCL communicator: ranks only
exchange their device timings (max over ranks) through a gloo (host)
process group.  Shard invariance -- every image's output is bit-identical
whichever rank (plan, stream) processes it -- is tested on one GPU in
tests/test_shard_gpu.py.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def partition(weights: Sequence[int], world: int) -> List[Tuple[int, int]]:
    """Contiguous [lo, hi) ranges, one per rank, with near-equal weight sums.

    Greedy prefix split at the ideal cumulative targets k * total / world;
    every rank gets a range (possibly empty when there are fewer images than
    ranks)."""
    n = len(weights)
    if world < 1:
        raise ValueError("world must be >= 1")
    total = float(sum(weights))
    bounds = [0]
    acc = 0.0
    i = 0
    for k in range(1, world):
        target = total * k / world
        while i < n and acc + weights[i] / 2.0 <= target:
            acc += weights[i]
            i += 1
        bounds.append(max(bounds[-1], i))
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def roi_weights(params, images) -> List[int]:
    """ROI block count of each image under `params` (host-only geometry)."""
    from . import geometry
    cache = {}
    out = []
    for im in images:
        key = (im.width, im.height)
        if key not in cache:
            cache[key] = geometry(params, im.width, im.height)["roi_blocks"]
        out.append(int(cache[key]))
    return out


def max_over_ranks(value: float) -> float:
    """Max of a per-rank scalar (e.g. elapsed ms) over the (gloo) process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
