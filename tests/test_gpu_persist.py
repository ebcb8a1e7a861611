"""Persistent single-launch CG solver (cg.cu, cg_persist_2048_kernel: FP32, L = 2048; opt-in with
BSCT_PERSIST=1, measured slower than the per-pass launches).  It runs the same pass-A / B / C tile
functions as the per-pass kernels, separated by grid barriers, with the Parseval partials summed
per column pair in the same order, so its iterates, residual history and breakdown flags must
equal the per-pass launches bit for bit (CG per slice); and it must match the FP64 oracle
CG at the FP32 CG tolerance of test_gpu_solvers (1e-4 for k <= 5)."""
import numpy as np
import pytest

from gpu_util import gpu_plan, rel_l2, to_dev, to_np
from oracle import solvers
from oracle.gram import gram_taps
from oracle.normal import apply_fft
from synth import CONFIGS
from synth.phantom import config_image

pytestmark = pytest.mark.gpu


def solve(bsct, plan, b, K, persist, monkeypatch, solver="cg"):
    import torch
    monkeypatch.setenv("BSCT_PERSIST", persist)
    B, N = b.shape[0], b.shape[1]
    x = torch.full((B, N, N), np.nan, device="cuda")
    hist = torch.zeros((B, K), dtype=torch.float64, device="cuda")
    flags = torch.zeros(B, dtype=torch.int32, device="cuda")
    bsct.cg_solve(plan, b, x, K, solver, resid_hist=hist, flags=flags)
    torch.cuda.synchronize()
    return x.cpu(), hist.cpu(), flags.cpu()


# N = 1024: full columns and 16-byte rows (config 4); 1000: 16-byte rows, ragged columns;
# 701: unaligned rows (scalar staging); 513: the smallest N with L = 2048
@pytest.mark.parametrize("N", [1024, 1000, 701, 513])
@pytest.mark.parametrize("B", [1, 3])
def test_persist_bitwise_per_pass(cuda_lib, monkeypatch, N, B):
    import torch
    cfg = CONFIGS[4].with_(N=N, n_angles=60, n_det=2 * N + 1, ellipse_scale=N / 64)
    plan, _ = gpu_plan(cuda_lib, cfg.geometry(), "f32", max_batch=B)
    torch.manual_seed(N + B)
    b = torch.rand((B, N, N), device="cuda")
    if B > 1:
        b[1] = 0  # rho_0 = 0: alpha = 0 every iteration, x stays 0 (the frozen-slice path)
    K = 6
    ref = solve(cuda_lib, plan, b, K, "0", monkeypatch)
    for _ in range(2):
        got = solve(cuda_lib, plan, b, K, "1", monkeypatch)
        for a, c in zip(ref, got):
            assert torch.equal(a, c)
    assert torch.isfinite(ref[0]).all()
    if B > 1:
        assert not ref[0][1].any()


@pytest.mark.parametrize("N,lam_y,zeta", [(1024, 0.5, 0.5), (600, 1.0, 1.0)])
def test_persist_vs_oracle(cuda_lib, monkeypatch, N, lam_y, zeta):
    """Config 4's geometry (lambda_y = 0.5, zeta = 0.5) at N = 1024 and a ragged N = 600, two
    slices, against oracle.solvers.cg from the same b = G c."""
    import torch
    cfg = CONFIGS[4].with_(N=N, n_angles=90, n_det=int(2 * N / lam_y) + 1, lambda_y=lam_y, zeta=zeta,
                           ellipse_scale=N / 64)
    g = cfg.geometry()
    T = gram_taps(g)
    B, K = 2, 5
    b = np.stack([apply_fft(T, config_image(cfg, s)) for s in range(B)])
    plan, _ = gpu_plan(cuda_lib, g, "f32", max_batch=B)
    x, h, f = solve(cuda_lib, plan, to_dev(b, "f32"), K, "1", monkeypatch)
    assert not f.any()
    for s in range(B):
        xr, hr = solvers.cg(T, b[s], K)
        assert rel_l2(x[s].double().numpy(), xr) < 1e-4
        assert rel_l2(h[s].numpy(), hr) < 1e-4


def test_persist_policy(cuda_lib, monkeypatch):
    """Default: the per-pass launches (3 per iteration + init + finish); BSCT_PERSIST=1: init, one
    cooperative launch for every iteration, finish."""
    import torch
    monkeypatch.setenv("BSCT_GRAPH", "0")
    N = 520
    cfg = CONFIGS[4].with_(N=N, n_angles=30, n_det=2 * N + 1, ellipse_scale=N / 64)
    plan, _ = gpu_plan(cuda_lib, cfg.geometry(), "f32", max_batch=6)
    K = 4
    for persist, launches in ((None, 3 * K + 2), ("1", 3)):
        if persist is None:
            monkeypatch.delenv("BSCT_PERSIST", raising=False)
        else:
            monkeypatch.setenv("BSCT_PERSIST", persist)
        for B in (1, 6):
            b = torch.rand((B, N, N), device="cuda")
            x = torch.empty_like(b)
            cuda_lib.cg_solve(plan, b, x, K, "cg")
            torch.cuda.synchronize()
            assert plan.launches == launches
