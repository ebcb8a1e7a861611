"""Multi-GPU plumbing over torch.distributed (NCCL on the GPU box, gloo in CPU tests).

Only where the path shards:
* slice_shard     -- config 5: contiguous blocks of slices per rank; no collective in the
                     data path (each rank back projects and solves its own slices).
* angle_shard /
  gram_build_sharded -- config 4: each rank builds the partial Gram filter over its angle
                     range (bsct_gram_build(angle_begin, angle_end), P:96-129 is a sum over
                     angles) and the partials are summed by one allreduce over NVLink.
* angle_shard_geometry /
  backproject_sharded -- one large slice: the back projection
                     b = H^T g is also a sum over angles, so each rank back projects
                     its angle range with a plan built on the sub-geometry and one allreduce of
                     the N^2 partial image (4 MB at N = 1024) sums them.
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
    _order_before_collective(stream)
    return allreduce_taps(taps, group)


def _order_before_collective(stream):
    """torch's NCCL collectives are ordered after work on torch's CURRENT stream only: when the
    library call ran on another stream, make the current stream wait for it (no host sync)."""
    if stream is None:
        return
    import torch
    torch.cuda.current_stream().wait_stream(stream)


def angle_shard_geometry(geom: dict, world: int, rank: int) -> tuple[dict, int, int]:
    """This rank's sub-geometry (angles[a0:a1], everything else unchanged) and [a0, a1)."""
    a0, a1 = angle_shard(len(geom["angles"]), world, rank)
    sub = dict(geom)
    sub["angles"] = list(geom["angles"])[a0:a1]
    return sub, a0, a1


def backproject_sharded(plan_shard, sino_shard, b, group=None, stream=None):
    """Full back projection b[B, N, N] of a sinogram whose angles are split over the ranks:
    this rank's partial H^T g over its angle range (plan_shard built on
    angle_shard_geometry(...)[0], sino_shard = sino[:, a0:a1, :]), then allreduce(SUM).
    plan_shard None (an empty angle range when world > n_angles) contributes zeros."""
    import torch.distributed as dist

    from . import backproject
    if plan_shard is None:
        b.zero_()
    else:
        backproject(plan_shard, sino_shard, b, stream=stream)
    _order_before_collective(stream)
    dist.all_reduce(b, op=dist.ReduceOp.SUM, group=group)
    return b
