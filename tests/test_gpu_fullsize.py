"""Parity at BASELINE.json's full config-5 size in the launch configuration bench.py times:
2048 slices of N = 512 in one bsct_reconstruct call (K4 v3 with 4 slices per CTA, the
FP32 warp-FFT CG passes at L = 1024, 50 CG iterations), checked on sampled outputs the
oracle can compute one by one:

* back projection: sampled pixels of the first, a middle and the last slice against
  oracle.backproject (1e-5 relative L2, north_star);
* CG: slices of the 2048-slice batch are bitwise equal to the same slices solved alone
  (B = 1; deterministic per-slice reductions, R20), and one slice meets the objective
  guard of R12 against the FP64 oracle CG.

Inputs: seeded uniform sinograms made on the device (the operators are linear; the
values do not change what is compared), with the checked slices copied to the host.
"""
import numpy as np
import pytest

from gpu_util import rel_l2, to_dev, to_np
from oracle import solvers
from oracle.backproject import backproject
from oracle.gram import gram_taps
from synth import CONFIGS

pytestmark = pytest.mark.gpu


def test_config5_full_batch(cuda_lib):
    import torch
    cfg = CONFIGS[5]
    g = cfg.geometry()
    N, n, M, B, K = cfg.N, cfg.n_angles, cfg.n_det, cfg.n_slices, cfg.iters
    assert B == 2048 and N == 512 and K == 50
    taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
    cuda_lib.gram_build(g, taps)
    plan = cuda_lib.plan_create(g, taps, max_batch=B)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5005)
    sino = torch.rand((B, n, M), device="cuda", generator=gen) * 0.4 + 0.1
    b = torch.empty((B, N, N), device="cuda")
    cuda_lib.backproject(plan, sino, b)
    x = torch.empty((B, N, N), device="cuda")
    cuda_lib.reconstruct(plan, sino, x, K, "cg")
    torch.cuda.synchronize()

    rng = np.random.default_rng(55)
    for s in (0, 1027, B - 1):
        k1 = np.concatenate([[0, 0, N - 1, N - 1], rng.integers(0, N, 196)])
        k2 = np.concatenate([[0, N - 1, 0, N - 1], rng.integers(0, N, 196)])
        ref = backproject(g, sino[s].double().cpu().numpy(), pixels=(k1, k2))
        assert rel_l2(to_np(b[s])[k1, k2], ref) < 1e-5, s

    # batched == single (bitwise), at both ends of the batch and in a ragged last SB group
    plan1 = cuda_lib.plan_create(g, taps, max_batch=1)
    for s in (0, 2046):
        x1 = torch.empty((1, N, N), device="cuda")
        cuda_lib.reconstruct(plan1, sino[s:s + 1].contiguous(), x1, K, "cg")
        torch.cuda.synchronize()
        assert torch.equal(x1[0], x[s]), s

    # R12 objective guard for one slice against the FP64 oracle (same right-hand side)
    T = gram_taps(g)
    bs = to_np(b[0])
    xk, _ = solvers.cg(T, bs, int(np.ceil(0.8 * K)))
    assert solvers.objective(T, bs, to_np(x[0])) <= solvers.objective(T, bs, xk)


def test_maximum_size_N2048(cuda_lib):
    """Largest supported FP32 slice (N = 2048: L = 4096 generic FFT passes; K4 v3 over 32 x 32
    tiles): taps, back projection (sampled pixels), normal apply (against the oracle's FFT
    apply), 2 CG iterations; then empty batches through every call (no-ops)."""
    import torch
    from oracle.gram import gram_taps
    from oracle.normal import apply_fft
    N, n, M = 2048, 16, 2 * 2048 + 1
    g = dict(N=N, lambda_x=1.0, angles=np.arange(n) * np.pi / n + 0.01, lambda_y=1.0, n_det=M, zeta=1.0)
    taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
    cuda_lib.gram_build(g, taps)
    T = gram_taps(g)
    assert rel_l2(to_np(taps), T) < 1e-5
    plan = cuda_lib.plan_create(g, taps, max_batch=1)
    assert plan.L == 4096
    rng = np.random.default_rng(2048)
    sino = rng.uniform(0, 1, (1, n, M))
    b = torch.empty((1, N, N), device="cuda")
    cuda_lib.backproject(plan, to_dev(sino, "f32"), b)
    k1, k2 = rng.integers(0, N, 100), rng.integers(0, N, 100)
    assert rel_l2(to_np(b[0])[k1, k2], backproject(g, sino[0], pixels=(k1, k2))) < 1e-5
    x = to_dev(rng.uniform(-1, 1, (1, N, N)), "f32")
    y = torch.empty_like(x)
    cuda_lib.normal_apply(plan, x, y)
    ref = apply_fft(T, to_np(x[0]))
    assert rel_l2(to_np(y[0]), ref) < 1e-5
    xs = torch.empty_like(b)
    cuda_lib.cg_solve(plan, b, xs, 2, "cg")
    xr, _ = solvers.cg(T, to_np(b[0]), 2)
    assert rel_l2(to_np(xs[0]), xr) < 1e-4
    # empty batch: every call is a no-op
    cuda_lib.backproject(plan, to_dev(sino[:0], "f32"), b[:0])
    cuda_lib.cg_solve(plan, b[:0], xs[:0], 2, "cg")
    cuda_lib.reconstruct(plan, to_dev(sino[:0], "f32"), xs[:0], 2, "cg")
