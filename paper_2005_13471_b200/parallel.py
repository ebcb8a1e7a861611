"""Multi-GPU plumbing over torch.distributed (NCCL on the GPU box, gloo in CPU tests).

Only where the path shards:
* slice_shard     -- config 5: contiguous blocks of slices per rank; no collective in the
                     data path (each rank back projects and solves its own slices).
* angle_shard /
  gram_build_sharded -- config 4: each rank builds the partial Gram filter over its angle
                     range (bsct_gram_build(angle_begin, angle_end), P:96-129 is a sum over
                     angles) and the partials are summed by one allreduce over NVLink.
"""
from __future__ import annotations


def shard(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return rank * n // world, (rank + 1) * n // world


def slice_shard(n_slices: int, world: int, rank: int) -> tuple[int, int]:
    return shard(n_slices, world, rank)


def angle_shard(n_angles: int, world: int, rank: int) -> tuple[int, int]:
    return shard(n_angles, world, rank)


def allreduce_taps(taps, group=None):
    """Sum the ranks' partial Gram filters in place (one collective)."""
    import torch.distributed as dist
    dist.all_reduce(taps, op=dist.ReduceOp.SUM, group=group)
    return taps


def gram_build_sharded(geom: dict, taps, group=None, stream=None):
    """Full Gram filter from angle shards: this rank's partial filter, then allreduce(SUM)."""
    import torch.distributed as dist

    from . import gram_build
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    a0, a1 = angle_shard(len(geom["angles"]), world, rank)
    gram_build(geom, taps, a0, a1, stream=stream)
    return allreduce_taps(taps, group)
