"""GPU parity of the solver loop (K6 + K5) vs oracle.solvers (north_star).

Tolerances: FP64 CG at config 1: 1e-6; steepest descent
and Landweber: 1e-3 at the configured iteration count; FP32 CG: 1e-4 for k <= 5 and a
convergence guard on the objective f(x) = 1/2 <x, Gx> - <b, x> (FP32 CG iterates are
chaotic, so per-iterate parity at K is not a property of any correct FP32 CG)."""
import numpy as np
import pytest

from gpu_util import geom, gpu_plan, rel_l2, to_dev, to_np, uniform
from oracle import solvers
from oracle.gram import gram_taps
from oracle.normal import apply_fft
from synth import CONFIGS
from synth.phantom import config_image

pytestmark = pytest.mark.gpu


def rhs(cfg, taps_ref, B=1):
    """b = G c for the config's phantom image(s) (seeded; oracle FP64 apply)."""
    return np.stack([apply_fft(taps_ref, config_image(cfg, s)) for s in range(B)])


def run(bsct, cfg, b, iters, solver, B=1):
    import torch
    g = cfg.geometry()
    plan, taps = gpu_plan(bsct, g, cfg.dtype, max_batch=B)
    x = torch.empty((B, cfg.N, cfg.N), dtype=taps.dtype, device="cuda")
    hist = torch.empty((B, iters), dtype=torch.float64, device="cuda")
    flags = torch.empty((B,), dtype=torch.int32, device="cuda")
    bsct.cg_solve(plan, to_dev(b, cfg.dtype), x, iters, solver, resid_hist=hist, flags=flags)
    torch.cuda.synchronize()
    assert not flags.any()
    return to_np(x), hist.cpu().numpy()


def test_cg_config1_fp64(cuda_lib):
    cfg = CONFIGS[1]
    T = gram_taps(cfg.geometry())
    b = rhs(cfg, T)
    x, h = run(cuda_lib, cfg, b, cfg.iters, "cg")
    xr, hr = solvers.cg(T, b[0], cfg.iters)
    assert rel_l2(x[0], xr) < 1e-6
    # ||r_k|| of CG is far more rounding-sensitive than x_k: early iterations only
    assert rel_l2(h[0][:8], hr[:8]) < 1e-6


@pytest.mark.parametrize("ci,solver", [(1, "sd"), (1, "landweber"), (2, "sd"), (2, "landweber"),
                                       (3, "sd"), (3, "landweber")])
def test_sd_landweber(cuda_lib, ci, solver):
    cfg = CONFIGS[ci]
    T = gram_taps(cfg.geometry())
    b = rhs(cfg, T)
    x, h = run(cuda_lib, cfg, b, cfg.iters, solver)
    xr, hr = (solvers.sd if solver == "sd" else solvers.landweber)(T, b[0], cfg.iters)
    assert rel_l2(x[0], xr) < 1e-3
    assert rel_l2(h[0], hr) < 1e-3


@pytest.mark.parametrize("ci", [2, 3])
def test_cg_fp32(cuda_lib, ci):
    cfg = CONFIGS[ci]
    T = gram_taps(cfg.geometry())
    b = rhs(cfg, T)
    x5, _ = run(cuda_lib, cfg, b, 5, "cg")
    xr5, _ = solvers.cg(T, b[0], 5)
    assert rel_l2(x5[0], xr5) < 1e-4
    K = cfg.iters
    x, h = run(cuda_lib, cfg, b, K, "cg")
    xk, _ = solvers.cg(T, b[0], int(np.ceil(0.8 * K)))
    assert solvers.objective(T, b[0], x[0]) <= solvers.objective(T, b[0], xk)


@pytest.mark.parametrize("solver", ["cg", "sd", "landweber"])
def test_fused_equals_unfused(cuda_lib, solver, monkeypatch):
    """The fused 3-launch iteration (cg.cu) against the 5-launch one (solver.cu)."""
    cfg = CONFIGS[2].with_(N=96, n_angles=60, n_det=137, ellipse_scale=1.5)
    T = gram_taps(cfg.geometry())
    b = rhs(cfg, T, B=2)
    xf, hf = run(cuda_lib, cfg, b, 8, solver, B=2)
    monkeypatch.setenv("BSCT_SOLVER_V1", "1")
    xu, hu = run(cuda_lib, cfg, b, 8, solver, B=2)
    assert rel_l2(xf, xu) < 1e-5
    assert rel_l2(hf, hu) < 1e-5


def test_batched_equals_single(cuda_lib):
    cfg = CONFIGS[2].with_(N=64, n_angles=60, n_det=91, ellipse_scale=1.0)
    T = gram_taps(cfg.geometry())
    b = rhs(cfg, T, B=3)
    xb, hb = run(cuda_lib, cfg, b, 12, "cg", B=3)
    for i in range(3):
        xs, hs = run(cuda_lib, cfg, b[i:i + 1], 12, "cg", B=1)
        assert np.array_equal(xs[0], xb[i])


def test_single_pixel_and_zero_rhs(cuda_lib):
    cfg = CONFIGS[1].with_(N=1, n_det=5)
    T = gram_taps(cfg.geometry())
    b = np.array([[[2.5]]])
    x, h = run(cuda_lib, cfg, b, 1, "cg")
    assert x[0, 0, 0] == pytest.approx(2.5 / T[0, 0], rel=1e-12)
    cfg = CONFIGS[1].with_(N=16, n_det=33)
    x, h = run(cuda_lib, cfg, np.zeros((1, 16, 16)), 4, "cg")
    assert not x.any() and not h.any()


def test_reconstruct_host_matches_device(cuda_lib):
    import torch
    cfg = CONFIGS[2].with_(N=64, n_angles=60, n_det=91, ellipse_scale=1.0)
    g = cfg.geometry()
    from synth.sinogram import config_sinogram
    sino = np.stack([config_sinogram(cfg, s) for s in range(2)]).astype(np.float32)
    plan, taps = gpu_plan(cuda_lib, g, "f32", max_batch=2)
    sh = torch.from_numpy(sino).pin_memory()
    xh = torch.empty((2, 64, 64), dtype=torch.float32).pin_memory()
    cuda_lib.reconstruct_host(plan, sh, xh, 10, "cg")
    sd = sh.cuda()
    b = torch.empty((2, 64, 64), device="cuda")
    cuda_lib.backproject(plan, sd, b)
    x = torch.empty_like(b)
    cuda_lib.cg_solve(plan, b, x, 10, "cg")
    torch.cuda.synchronize()
    assert torch.equal(x.cpu(), xh)


@pytest.mark.parametrize("N", [129, 200, 256, 257, 300, 512, 700, 701])
@pytest.mark.parametrize("solver", ["cg", "sd", "landweber"])
def test_warp_fft_passes_equal_generic(cuda_lib, N, solver, monkeypatch):
    """FP32 warp-FFT passes (fft32.cuh; L = 512, 1024, 2048: passes A, B, C) against the
    generic block-FFT passes, ragged N (odd N exercises the unaligned staging path), B = 2."""
    cfg = CONFIGS[3].with_(N=N, n_angles=90, n_det=2 * N + 1, ellipse_scale=N / 64)
    T = gram_taps(cfg.geometry())
    b = rhs(cfg, T, B=2)
    # FP32 CG amplifies rounding differences (R12): 5 iterations at 1e-4 as in test_cg_fp32
    K, tl = (5, 1e-4) if solver == "cg" else (6, 1e-5)
    xw, hw = run(cuda_lib, cfg, b, K, solver, B=2)
    monkeypatch.setenv("BSCT_PASSB_V1", "1")
    monkeypatch.setenv("BSCT_PASSC_V1", "1")
    xg, hg = run(cuda_lib, cfg, b, K, solver, B=2)
    assert rel_l2(xw, xg) < tl
    assert rel_l2(hw, hg) < tl
    xr, _ = {"cg": solvers.cg, "sd": solvers.sd, "landweber": solvers.landweber}[solver](T, b[1], K)
    assert rel_l2(xw[1], xr) < 1e-4


@pytest.mark.parametrize("chunk,overlap", [("0", "0"), ("2", "0"), ("2", "1"), ("3", "1")])
@pytest.mark.parametrize("solver", ["cg", "landweber"])
def test_reconstruct_pipeline_equals_sequence(cuda_lib, chunk, overlap, solver, monkeypatch):
    """bsct_reconstruct (slice chunks: back projection on the plan's stream overlapping the
    solves) is bitwise identical to bsct_backproject + bsct_cg_solve; resid/flags offsets."""
    import torch
    from synth.sinogram import config_sinogram
    monkeypatch.setenv("BSCT_PIPE_CHUNK", chunk)
    monkeypatch.setenv("BSCT_PIPE_OVERLAP", overlap)
    cfg = CONFIGS[2].with_(N=64, n_angles=60, n_det=91, ellipse_scale=1.0)
    g = cfg.geometry()
    B = 5
    sino = np.stack([config_sinogram(cfg, s) for s in range(B)]).astype(np.float32)
    plan, taps = gpu_plan(cuda_lib, g, "f32", max_batch=B)
    sd = to_dev(sino, "f32")
    x = torch.empty((B, 64, 64), device="cuda")
    h = torch.empty((B, 7), dtype=torch.float64, device="cuda")
    cuda_lib.reconstruct(plan, sd, x, 7, solver, resid_hist=h)
    b = torch.empty_like(x)
    cuda_lib.backproject(plan, sd, b)
    x2 = torch.empty_like(x)
    h2 = torch.empty_like(h)
    cuda_lib.cg_solve(plan, b, x2, 7, solver, resid_hist=h2)
    torch.cuda.synchronize()
    assert torch.equal(x, x2)
    assert torch.equal(h, h2)
    xh = torch.empty((B, 64, 64), dtype=torch.float32).pin_memory()
    cuda_lib.reconstruct_host(plan, torch.from_numpy(sino).pin_memory(), xh, 7, solver)
    assert torch.equal(xh, x.cpu())


@pytest.mark.parametrize("ci,iters,tl", [(1, 20, 1e-9), (2, 50, 1e-4), (3, 100, 1e-3)])  # 1e-3: north_star reconstructions
def test_chebyshev(cuda_lib, ci, iters, tl):
    """NEXT-4: Chebyshev semi-iteration vs the FP64 oracle at the config's iteration count.  No
    inner products, so unlike FP32 CG (R12) the FP32 iterates keep parity with FP64; the
    interval is [lambda_max / 1e3, lambda_max], lambda_max = max of the embedding spectrum."""
    import torch
    cfg = CONFIGS[ci]
    T = gram_taps(cfg.geometry())
    b = rhs(cfg, T)
    lmax = 1.0 / solvers.landweber_tau(T)
    lmin = lmax / 1e3
    g = cfg.geometry()
    plan, taps = gpu_plan(cuda_lib, g, cfg.dtype, max_batch=1)
    x = torch.empty((1, cfg.N, cfg.N), dtype=taps.dtype, device="cuda")
    h = torch.empty((1, iters), dtype=torch.float64, device="cuda")
    cuda_lib.chebyshev_solve(plan, to_dev(b, cfg.dtype), x, iters, lmin, lmax, resid_hist=h)
    torch.cuda.synchronize()
    xr, hr = solvers.chebyshev(T, b[0], iters, lmin, lmax)
    assert rel_l2(to_np(x[0]), xr) < tl
    assert rel_l2(h.cpu().numpy()[0], hr) < tl
    # the plan's own spectrum bound (lambda_max <= 0) gives the same iterate up to FP rounding
    x2 = torch.empty_like(x)
    cuda_lib.chebyshev_solve(plan, to_dev(b, cfg.dtype), x2, iters, lmin)
    torch.cuda.synchronize()
    assert rel_l2(to_np(x2[0]), xr) < 10 * tl
    with pytest.raises(cuda_lib.BsctError):
        cuda_lib.chebyshev_solve(plan, to_dev(b, cfg.dtype), x2, iters, lmax * 2, lmax)


@pytest.mark.parametrize("N,dt", [(1, "f32"), (16, "f64"), (64, "f64"), (100, "f32"), (128, "f32"), (200, "f32"),
                                  (256, "f32"), (128, "f64")])
@pytest.mark.parametrize("solver", ["cg", "sd", "landweber"])
def test_onchip_cluster_solver(cuda_lib, N, dt, solver, monkeypatch):
    """NEXT-2: the cluster-resident solver loop (onchip.cu, one thread-block cluster of 1-8 CTAs
    per slice, T1 distributed over the CTAs' shared memory) against the fused multi-launch path
    (BSCT_ONCHIP=0) and, for CG, the FP64 oracle; B = 3 with distinct right-hand sides."""
    cfg = CONFIGS[2].with_(N=N, n_angles=48, n_det=2 * N + 3, ellipse_scale=max(N, 8) / 64, dtype=dt)
    T = gram_taps(cfg.geometry())
    b = rhs(cfg, T, B=3)
    K = 5 if solver == "cg" else 6  # FP32 CG iterates keep 1e-4 parity for k <= 5 only
    monkeypatch.setenv("BSCT_ONCHIP", "1")
    xo, ho = run(cuda_lib, cfg, b, K, solver, B=3)
    monkeypatch.setenv("BSCT_ONCHIP", "0")
    xf, hf = run(cuda_lib, cfg, b, K, solver, B=3)
    tl = 1e-10 if dt == "f64" else (1e-4 if solver == "cg" else 1e-5)
    assert rel_l2(xo, xf) < tl
    assert rel_l2(ho, hf) < tl
    if solver == "cg":
        xr, _ = solvers.cg(T, b[2], K)
        assert rel_l2(xo[2], xr) < (1e-9 if dt == "f64" else 1e-4)


def test_bulk_staging_equals_cp_async(cuda_lib, monkeypatch):
    """Pass C's T1 tile staged by bulk (TMA) copies (BSCT_BULK=1) equals the cp.async staging."""
    cfg = CONFIGS[3].with_(N=512, n_angles=60, n_det=725, ellipse_scale=8.0)
    T = gram_taps(cfg.geometry())
    b = rhs(cfg, T, B=2)
    monkeypatch.setenv("BSCT_BULK", "1")
    xb, hb = run(cuda_lib, cfg, b, 4, "cg", B=2)
    monkeypatch.setenv("BSCT_BULK", "0")
    xc, hc = run(cuda_lib, cfg, b, 4, "cg", B=2)
    assert np.array_equal(xb, xc) and np.array_equal(hb, hc)


@pytest.mark.parametrize("solver", ["cg", "sd", "landweber"])
def test_graph_replay_equals_launches(cuda_lib, solver, monkeypatch):
    """Small solves are captured into a CUDA graph and replayed (api.cu solve_t): bitwise equal
    to plain launches, on first capture and on replay with new data in the same buffers."""
    import torch
    cfg = CONFIGS[2].with_(N=64, n_angles=40, n_det=131, ellipse_scale=1.0)
    g = cfg.geometry()
    T = gram_taps(g)
    b = rhs(cfg, T, B=2)
    plan, taps = gpu_plan(cuda_lib, g, "f32", max_batch=2)
    bd = to_dev(b, "f32")
    xs = []
    for mode in ("1", "1", "0"):  # capture, replay, plain launches
        monkeypatch.setenv("BSCT_GRAPH", mode)
        x = torch.zeros((2, 64, 64), device="cuda") if not xs else xs[0][0]
        h = torch.zeros((2, 7), dtype=torch.float64, device="cuda") if not xs else xs[0][1]
        cuda_lib.cg_solve(plan, bd, x, 7, solver, resid_hist=h)
        torch.cuda.synchronize()
        xs.append((x, h, x.clone(), h.clone()))
        bd.mul_(1.0)  # same data, same buffers
    assert torch.equal(xs[0][2], xs[1][2]) and torch.equal(xs[0][3], xs[1][3])
    assert torch.equal(xs[0][2], xs[2][2]) and torch.equal(xs[0][3], xs[2][3])
    xr, _ = {"cg": solvers.cg, "sd": solvers.sd, "landweber": solvers.landweber}[solver](T, b[1], 7)
    # FP32 CG beyond k = 5 drifts from FP64 (R12): north_star's 1e-3; SD / Landweber keep 1e-4
    assert rel_l2(xs[0][2].double().cpu().numpy()[1], xr) < (1e-3 if solver == "cg" else 1e-4)
