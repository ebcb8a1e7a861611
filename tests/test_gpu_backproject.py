"""GPU parity, part (b): correction filter (K3, Eq.(5)) and back projection H^T g^
(K4) vs oracle.backproject; forward projection (K7, Eq.(3)-(4)) vs
oracle.forward; the exact-recovery property of P:140 through the CUDA path."""
import numpy as np
import pytest

from gpu_util import geom, gpu_plan, rel_l2, to_dev, to_np, tol, uniform
from oracle.backproject import H_CORR, backproject, corrected_row, interpolation_degree
from oracle.forward import forward
from synth import CONFIGS
from synth.sinogram import config_sinogram, random_sinogram

pytestmark = pytest.mark.gpu


def gpu_bp(bsct, g, dt, sino):
    import torch
    B = sino.shape[0]
    plan, taps = gpu_plan(bsct, g, dt, max_batch=B)
    b = torch.empty((B, g["N"], g["N"]), dtype=taps.dtype, device="cuda")
    bsct.backproject(plan, to_dev(sino, dt), b)
    return plan, to_np(b)


@pytest.mark.parametrize("zeta,ly,dt", [(0.0, 1.0, "f32"), (1.0, 1.0, "f64"), (1.5, 1.0, "f32"),
                                        (0.5, 0.5, "f32"), (0.7, 1.3, "f64")])
def test_correction_filter(cuda_lib, zeta, ly, dt):
    import torch
    n, M = 12, 37
    g = geom(6, uniform(n), M, lambda_y=ly, zeta=zeta)
    sino = random_sinogram(3, 2, n, M)
    plan, _ = gpu_plan(cuda_lib, g, dt, max_batch=2)
    gt = torch.empty((2, n, M + 2 * H_CORR), dtype=plan.dtype, device="cuda")
    cuda_lib.correction_filter(plan, to_dev(sino, dt), gt)
    got = to_np(gt)
    for bi in range(2):
        for a, t in enumerate(g["angles"]):
            ref = corrected_row(sino[bi, a], interpolation_degree(g, t))
            assert rel_l2(got[bi, a], ref) < tol(dt)


@pytest.mark.parametrize("M,B,dt", [(5, 1, "f32"), (38, 5, "f32"), (39, 4, "f64"), (40, 7, "f32"), (53, 9, "f64"),
                                    (725, 6, "f32"), (725, 3, "f64")])
def test_correction_filter_tails(cuda_lib, M, B, dt):
    """K3 v2 thread/CTA tiling (4 outputs per thread, 4 rows per CTA): every residue of M + 50 mod 4,
    ragged last CTAs (B mod 4 != 0) and the config-5 row length, each row against the oracle."""
    import torch
    n = 6
    g = geom(6, uniform(n), M, lambda_y=1.0, zeta=1.0)
    sino = random_sinogram(M + B, B, n, M)
    plan, _ = gpu_plan(cuda_lib, g, dt, max_batch=B)
    gt = torch.full((B, n, M + 2 * H_CORR), float("nan"), dtype=plan.dtype, device="cuda")
    cuda_lib.correction_filter(plan, to_dev(sino, dt), gt)
    got = to_np(gt)
    assert np.isfinite(got).all()
    for bi in range(B):
        for a, t in enumerate(g["angles"]):
            ref = corrected_row(sino[bi, a], interpolation_degree(g, t))
            assert rel_l2(got[bi, a], ref) < tol(dt)


@pytest.mark.parametrize("N,n,M,ly,zeta,dt,B", [
    (1, 3, 5, 1.0, 0.0, "f32", 1), (4, 8, 9, 1.0, 1.0, "f64", 2), (7, 11, 15, 0.5, 0.5, "f32", 2),
    (16, 24, 33, 1.0, 0.0, "f32", 1), (16, 24, 23, 1.3, 1.7, "f64", 1), (33, 36, 49, 1.0, 1.5, "f32", 2),
    (20, 12, 121, 0.25, 0.25, "f32", 2)])  # fine detector: K4 v2 tables exceed smem -> K4 v1
def test_small_full(cuda_lib, N, n, M, ly, zeta, dt, B):
    g = geom(N, uniform(n), M, lambda_y=ly, zeta=zeta)
    sino = random_sinogram(N + n, B, n, M)
    _, b = gpu_bp(cuda_lib, g, dt, sino)
    for i in range(B):
        assert rel_l2(b[i], backproject(g, sino[i])) < tol(dt)


@pytest.mark.parametrize("ci", [1, 2, 4])
def test_v2_equals_v1(cuda_lib, ci, monkeypatch):
    """K4 v2 (per-tile piecewise-polynomial tables) against K4 v1 (direct per-sample
    evaluation) on the same device inputs; both are checked against the oracle elsewhere."""
    cfg = CONFIGS[ci]
    g = cfg.geometry()
    sino = config_sinogram(cfg)[None]
    _, b2 = gpu_bp(cuda_lib, g, cfg.dtype, sino)
    monkeypatch.setenv("BSCT_BP_V1", "1")
    _, b1 = gpu_bp(cuda_lib, g, cfg.dtype, sino)
    assert rel_l2(b2, b1) < (1e-12 if cfg.dtype == "f64" else 2e-6)


def test_config1_full(cuda_lib):
    cfg = CONFIGS[1]
    g = cfg.geometry()
    sino = config_sinogram(cfg)[None]
    _, b = gpu_bp(cuda_lib, g, cfg.dtype, sino)
    assert rel_l2(b[0], backproject(g, sino[0])) < tol(cfg.dtype)


@pytest.mark.parametrize("ci", [2, 3, 4, 5])
def test_config_sampled(cuda_lib, ci):
    """Full-size back projection, 400 sampled pixels (incl. corners) checked one by one."""
    cfg = CONFIGS[ci]
    g = cfg.geometry()
    sino = config_sinogram(cfg)[None]
    _, b = gpu_bp(cuda_lib, g, cfg.dtype, sino)
    N = cfg.N
    rng = np.random.default_rng(ci)
    k1 = np.concatenate([[0, 0, N - 1, N - 1, N // 2], rng.integers(0, N, 395)])
    k2 = np.concatenate([[0, N - 1, 0, N - 1, N // 2], rng.integers(0, N, 395)])
    ref = backproject(g, sino[0], pixels=(k1, k2))
    assert rel_l2(b[0][k1, k2], ref) < 1e-5


@pytest.mark.parametrize("N,n,M,ly,zeta,lx,dt", [
    (1, 4, 7, 0.75, 0.0, 1.0, "f64"), (5, 7, 13, 0.8, 0.0, 1.0, "f32"), (6, 9, 21, 1.0, 1.0, 1.0, "f64"),
    (9, 13, 31, 0.5, 0.4, 0.5, "f32"), (24, 30, 49, 1.0, 1.5, 1.0, "f32")])
def test_forward(cuda_lib, N, n, M, ly, zeta, lx, dt):
    import torch
    g = geom(N, uniform(n) + 0.01, M, lambda_y=ly, zeta=zeta, lambda_x=lx)
    c = np.random.default_rng(N).uniform(-1, 1, (2, N, N))
    plan, taps = gpu_plan(cuda_lib, g, dt, max_batch=2)
    s = torch.empty((2, n, M), dtype=taps.dtype, device="cuda")
    cuda_lib.forward_project(plan, to_dev(c, dt), s)
    for i in range(2):
        assert rel_l2(to_np(s[i]), forward(g, c[i])) < tol(dt)


def test_forward_config_sparse(cuda_lib):
    """Config-5 geometry, sparse image (the oracle sums nonzero pixels only)."""
    import torch
    cfg = CONFIGS[5]
    g = cfg.geometry()
    N = cfg.N
    c = np.zeros((N, N))
    rng = np.random.default_rng(5)
    c[rng.integers(0, N, 40), rng.integers(0, N, 40)] = rng.uniform(0, 1, 40)
    plan, taps = gpu_plan(cuda_lib, g, "f32")
    s = torch.empty((1, cfg.n_angles, cfg.n_det), device="cuda")
    cuda_lib.forward_project(plan, to_dev(c[None], "f32"), s)
    assert rel_l2(to_np(s[0]), forward(g, c)) < 1e-5


@pytest.mark.parametrize("zeta", [0.0, 1.0])
def test_exact_recovery_on_device(cuda_lib, zeta):
    """BP(forward(c)) = G c at angles {0, pi/2}, lambda_y = lambda_x, all on the GPU."""
    import torch
    N = 20
    g = geom(N, [0.0, np.pi / 2], 2 * N + 9, zeta=zeta)
    plan, taps = gpu_plan(cuda_lib, g, "f64", max_batch=1)
    c = to_dev(np.random.default_rng(4).standard_normal((1, N, N)), "f64")
    s = torch.empty((1, 2, 2 * N + 9), dtype=torch.float64, device="cuda")
    cuda_lib.forward_project(plan, c, s)
    b = torch.empty_like(c)
    cuda_lib.backproject(plan, s, b)
    y = torch.empty_like(c)
    cuda_lib.normal_apply(plan, c, y)
    assert rel_l2(to_np(b), to_np(y)) < 1e-12


@pytest.mark.parametrize("sb", ["1", "2", "4"])
@pytest.mark.parametrize("ci,B", [(2, 5), (3, 3), (4, 2)])
def test_v3_slices_per_cta(cuda_lib, ci, B, sb, monkeypatch):
    """K4 v3 (SB slices per CTA sharing each pixel's locate; ragged batch when B % SB != 0)
    against K4 v2 on the same device inputs, and one slice against the oracle (sampled)."""
    cfg = CONFIGS[ci]
    g = cfg.geometry()
    rng = np.random.default_rng(ci * 10 + B)
    sino = config_sinogram(cfg)[None] * rng.uniform(0.5, 1.5, (B, 1, 1))
    sino = sino + 0.01 * rng.standard_normal(sino.shape)
    monkeypatch.setenv("BSCT_BP_SB", sb)
    _, b3 = gpu_bp(cuda_lib, g, "f32", sino)
    monkeypatch.setenv("BSCT_BP_V2", "1")
    _, b2 = gpu_bp(cuda_lib, g, "f32", sino)
    for i in range(B):
        assert rel_l2(b3[i], b2[i]) < 2e-6
    N = cfg.N
    k1, k2 = rng.integers(0, N, 200), rng.integers(0, N, 200)
    ref = backproject(g, sino[B - 1], pixels=(k1, k2))
    assert rel_l2(b3[B - 1][k1, k2], ref) < 1e-5


def test_angle_sharded_backprojection(cuda_lib):
    """the back projection of one large slice split over angle shards (plans on
    parallel.angle_shard_geometry sub-geometries) sums to the whole-geometry back projection;
    parallel.backproject_sharded end to end on a one-rank NCCL group; sampled pixels of the
    sum against the oracle."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2005_13471_b200.parallel import angle_shard_geometry, backproject_sharded
    N, n, M = 300, 90, 425
    g = dict(N=N, lambda_x=1.0, angles=list(np.arange(n) * np.pi / n + 0.02), lambda_y=1.0, n_det=M, zeta=1.0)
    taps = torch.zeros((2 * N - 1, 2 * N - 1), device="cuda")
    taps[N - 1, N - 1] = 1.0  # the back projection does not use the filter
    rng = np.random.default_rng(66)
    sino = rng.uniform(0, 1, (1, n, M))
    sd = to_dev(sino, "f32")
    full = torch.empty((1, N, N), device="cuda")
    cuda_lib.backproject(cuda_lib.plan_create(g, taps, max_batch=1), sd, full)
    acc = torch.zeros_like(full)
    part = torch.empty_like(full)
    for r in range(3):
        sub, a0, a1 = angle_shard_geometry(g, 3, r)
        cuda_lib.backproject(cuda_lib.plan_create(sub, taps, max_batch=1), sd[:, a0:a1].contiguous(), part)
        acc += part
    torch.cuda.synchronize()
    assert rel_l2(to_np(acc), to_np(full)) < 1e-6
    k1, k2 = rng.integers(0, N, 60), rng.integers(0, N, 60)
    assert rel_l2(to_np(acc[0])[k1, k2], backproject(g, sino[0], pixels=(k1, k2))) < 1e-5
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        sub, a0, a1 = angle_shard_geometry(g, 1, 0)
        out = torch.empty_like(full)
        backproject_sharded(cuda_lib.plan_create(sub, taps, max_batch=1), sd[:, a0:a1].contiguous(), out)
        torch.cuda.synchronize()
        assert torch.equal(out, full)
    finally:
        dist.destroy_process_group()


def test_two_devices_one_process(cuda_lib):
    """Per-device state (the correction filter q in __constant__ memory, the library memory pool,
    the cached angle sets) must exist on every device a process uses: the same back projection and
    Gram filter on device 0 and device 1 agree bitwise.  Needs two GPUs (skipped otherwise; the
    round's GPU runs have one)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    N, n, M = 64, 40, 101
    g = dict(N=N, lambda_x=1.0, angles=np.arange(n) * np.pi / n + 0.03, lambda_y=1.0, n_det=M, zeta=1.0)
    sino = np.random.default_rng(3).uniform(0, 1, (1, n, M))
    outs = []
    for d in (0, 1, 0):
        with torch.cuda.device(d):
            taps = torch.empty((2 * N - 1, 2 * N - 1), device=f"cuda:{d}")
            cuda_lib.gram_build(g, taps)
            plan = cuda_lib.plan_create(g, taps, max_batch=1)
            b = torch.empty((1, N, N), device=f"cuda:{d}")
            cuda_lib.backproject(plan, torch.as_tensor(sino, dtype=torch.float32, device=f"cuda:{d}"), b)
            torch.cuda.synchronize(d)
            outs.append((taps.cpu(), b.cpu()))
    for t, b in outs[1:]:
        assert torch.equal(t, outs[0][0]) and torch.equal(b, outs[0][1])


@pytest.mark.parametrize("N,n,M,zeta,lx,B", [(512, 360, 725, 1.0, 1.0, 130), (100, 60, 151, 1.0, 1.0, 3),
                                             (257, 90, 401, 1.5, 1.0, 5), (64, 32, 101, 0.0, 1.0, 2),
                                             (129, 45, 181, 1.0, 0.8, 129), (33, 30, 51, 1.0, 1.0, 1)])
def test_bp_tensor_core_equals_cuda_core(cuda_lib, N, n, M, zeta, lx, B, monkeypatch):
    """K4 v4 (tcgen05 tensor cores, 3xTF32, bp_tc.cu) against K4 v3 (FP32 CUDA cores) on the same
    sinograms: ragged pixel tiles (N not a multiple of 8 / 16), slice counts around the 128-slice
    MMA width, lambda_x != 1, no blur; and sampled pixels against the FP64 oracle."""
    import torch
    rng = np.random.default_rng(N + B)
    ang = np.arange(n) * np.pi / n + 0.013
    g = dict(N=N, lambda_x=lx, angles=ang, lambda_y=1.0, n_det=M, zeta=zeta)
    sino = rng.uniform(-1, 1, (B, n, M))
    sd = to_dev(sino, "f32")
    taps = torch.zeros((2 * N - 1, 2 * N - 1), device="cuda")
    taps[N - 1, N - 1] = 1.0  # the back projection does not read the filter
    out = {}
    for v3 in ("0", "1"):
        monkeypatch.setenv("BSCT_BP_V3", v3)
        plan = cuda_lib.plan_create(g, taps, max_batch=B)
        b = torch.empty((B, N, N), device="cuda")
        cuda_lib.backproject(plan, sd, b)
        torch.cuda.synchronize()
        out[v3] = to_np(b)
    assert rel_l2(out["0"], out["1"]) < 5e-6
    k1, k2 = rng.integers(0, N, 80), rng.integers(0, N, 80)
    assert rel_l2(out["0"][B - 1][k1, k2], backproject(g, sino[B - 1], pixels=(k1, k2))) < 1e-5
