"""World-size-2 gloo tests (CPU) of the multi-GPU plumbing: slice shards cover every slice
once, angle-sharded partial Gram filters allreduced with the product's collective equal the
full filter, and angle-sharded partial back projections allreduced equal the
full back projection (partials computed by the oracle here, by K1 / K4 on the GPU box)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_13471_b200.parallel import allreduce_taps, angle_shard, angle_shard_geometry, slice_shard


def test_shards_partition():
    for n in (1, 7, 360, 2048):
        for world in (1, 2, 3, 4, 8):
            blocks = [slice_shard(n, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        slice_shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.gram import gram_taps
    g = dict(N=12, lambda_x=1.0, angles=np.arange(30) * np.pi / 30, lambda_y=0.5, n_det=49, zeta=0.5)
    a0, a1 = angle_shard(30, world, rank)
    part = torch.tensor(gram_taps(g, a0, a1))
    allreduce_taps(part)
    if rank == 0:
        out.put(part.numpy())
    # slice shards: gather the covered slice ids
    lo, hi = slice_shard(2048, world, rank)
    t = torch.zeros(2048, dtype=torch.int64)
    t[lo:hi] = 1
    dist.all_reduce(t)
    if rank == 0:
        out.put(t.numpy())
    dist.destroy_process_group()


def test_gloo_angle_shards_allreduce():
    from oracle.gram import gram_taps
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    taps = q.get(timeout=120)
    cover = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = dict(N=12, lambda_x=1.0, angles=np.arange(30) * np.pi / 30, lambda_y=0.5, n_det=49, zeta=0.5)
    assert np.abs(taps - gram_taps(g)).max() < 1e-13
    assert (cover == 1).all()


G6 = dict(N=10, lambda_x=1.0, angles=list(np.arange(25) * np.pi / 25 + 0.05), lambda_y=0.75, n_det=31, zeta=1.0)


def _bp_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.backproject import backproject
    sino = np.random.default_rng(6).uniform(0, 1, (25, 31))
    sub, a0, a1 = angle_shard_geometry(G6, world, rank)
    assert len(sub["angles"]) == a1 - a0 and sub["N"] == G6["N"]
    part = torch.tensor(backproject(sub, sino[a0:a1]))
    dist.all_reduce(part)  # the collective of parallel.backproject_sharded
    if rank == 0:
        out.put(part.numpy())
    dist.destroy_process_group()


def test_gloo_angle_sharded_backprojection():
    from oracle.backproject import backproject
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    b = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sino = np.random.default_rng(6).uniform(0, 1, (25, 31))
    ref = backproject(G6, sino)
    assert np.abs(b - ref).max() < 1e-12 * np.abs(ref).max()
