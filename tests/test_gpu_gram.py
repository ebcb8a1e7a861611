"""GPU parity, part (a): Gram filter taps (K0 tables + K1) vs oracle.gram."""
import numpy as np
import pytest

from gpu_util import geom, gpu_taps, rel_l2, to_np, tol, uniform
from oracle.gram import gram_taps, gram_taps_at
from synth import CONFIGS

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,n,zeta,lx,dt", [
    (1, 1, 0.0, 1.0, "f32"), (2, 3, 0.5, 1.0, "f32"), (5, 7, 0.0, 1.0, "f32"), (13, 24, 1.0, 0.7, "f32"),
    (13, 24, 1.0, 1.0, "f64"), (33, 90, 1.5, 1.0, "f32"), (40, 36, 0.0, 1.0, "f64"), (17, 5, 2.5, 1.3, "f32")])
def test_small_geometries(cuda_lib, N, n, zeta, lx, dt):
    g = geom(N, uniform(n), 2 * N + 1, zeta=zeta, lambda_x=lx)
    G = to_np(gpu_taps(cuda_lib, g, dt))
    ref = gram_taps(g)
    assert rel_l2(G, ref) < tol(dt)
    assert np.abs(G - ref).max() < 10 * tol(dt) * np.abs(ref).max()
    assert np.array_equal(G, G[::-1, ::-1])          # G[k] = G[-k] bitwise (G symmetric)


def test_irregular_angles(cuda_lib):
    rng = np.random.default_rng(11)
    ang = rng.uniform(-3.0, 7.0, 29)                   # unsorted, outside [0, pi)
    g = geom(21, ang, 45, zeta=0.8)
    assert rel_l2(to_np(gpu_taps(cuda_lib, g, "f32")), gram_taps(g)) < 1e-5


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_clustered_angles(cuda_lib, dt):
    """Angle sets packed into a narrow wedge (an angle shard of config 4, repeated views): K1 sizes
    its central tile levels by the angular density, not by n; the taps still equal the oracle's."""
    wedge = 0.4 + np.arange(120) * (np.pi / 8 / 120)   # 120 angles in a pi/8 wedge
    repeated = np.concatenate([np.full(60, 1.1), [0.0, 2.0, 2.9]])
    for ang in (wedge, repeated, np.concatenate([wedge, wedge + np.pi])):   # the last wraps mod pi
        g = geom(48, ang, 97, zeta=1.0)
        G = to_np(gpu_taps(cuda_lib, g, dt))
        assert rel_l2(G, gram_taps(g)) < tol(dt)
        assert np.array_equal(G, G[::-1, ::-1])


def test_axis_and_45deg(cuda_lib):
    g = geom(6, [0.0, np.pi / 2, np.pi / 4], 13, zeta=0.0)
    assert rel_l2(to_np(gpu_taps(cuda_lib, g, "f64")), gram_taps(g)) < 1e-12


@pytest.mark.parametrize("ci", [1, 2, 3])
def test_config_full(cuda_lib, ci):
    cfg = CONFIGS[ci]
    g = cfg.geometry()
    G = to_np(gpu_taps(cuda_lib, g, cfg.dtype))
    ref = gram_taps(g)
    assert rel_l2(G, ref) < tol(cfg.dtype)


def test_config4_sampled(cuda_lib):
    """N = 1024, 720 angles, lambda_y = 0.5, zeta = 0.5 (BJ:configs[4]): every tap of the
    central 65 x 65 block plus 4000 random taps, against the oracle tap by tap."""
    cfg = CONFIGS[4]
    g = cfg.geometry()
    G = to_np(gpu_taps(cuda_lib, g, cfg.dtype))
    N = cfg.N
    rng = np.random.default_rng(12)
    c = np.arange(-32, 33)
    a = np.concatenate([np.repeat(c, c.size), rng.integers(-(N - 1), N, 4000)])
    b = np.concatenate([np.tile(c, c.size), rng.integers(-(N - 1), N, 4000)])
    ref = gram_taps_at(g, a, b)
    got = G[a + N - 1, b + N - 1]
    assert rel_l2(got, ref) < 1e-5


@pytest.mark.parametrize("ci", [2, 4])
def test_window_equals_dense(cuda_lib, ci, monkeypatch):
    """Windowed K1 (angle window per tap) against the dense angle loop."""
    g = CONFIGS[ci].geometry()
    win = to_np(gpu_taps(cuda_lib, g, "f32"))
    monkeypatch.setenv("BSCT_GRAM_DENSE", "1")
    dense = to_np(gpu_taps(cuda_lib, g, "f32"))
    assert rel_l2(win, dense) < 1e-6
    assert np.array_equal(win == 0, dense == 0)


def test_angle_shards_sum(cuda_lib):
    """BJ:configs[4]: angle-sharded partial filters sum to the full filter."""
    import torch
    g = geom(64, uniform(90), 129, zeta=0.5, lambda_y=0.5)
    full = gpu_taps(cuda_lib, g, "f32")
    parts = torch.zeros_like(full)
    tmp = torch.empty_like(full)
    for a0, a1 in ((0, 23), (23, 45), (45, 90)):
        cuda_lib.gram_build(g, tmp, a0, a1)
        parts += tmp
    assert rel_l2(to_np(parts), to_np(full)) < 1e-6
    cuda_lib.gram_build(g, tmp, 5, 5)                # empty shard -> zeros
    assert not tmp.any()


def test_gram_build_sharded_nccl(cuda_lib):
    """parallel.gram_build_sharded end to end on a one-rank NCCL group, the build queued on a
    non-current stream (the allreduce must be ordered after it), against the oracle; the
    angle-shard arithmetic over 4 ranks is covered by tests/test_parallel_gloo.py."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2005_13471_b200.parallel import gram_build_sharded
    g = geom(96, uniform(120), 193, zeta=0.5, lambda_y=0.5)
    ref = gram_taps(g)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        side = torch.cuda.Stream()
        for _ in range(3):
            taps = torch.full((191, 191), float("nan"), device="cuda")
            gram_build_sharded(g, taps, stream=side)
            torch.cuda.synchronize()
            assert rel_l2(to_np(taps), ref) < 1e-5
    finally:
        dist.destroy_process_group()
