"""GPU parity, part (c): filter spectrum (K2) and normal operator y = G x (K5) vs
oracle.normal, FP32 at 1e-5 relative L2 (north_star), FP64 at 1e-10 (R19)."""
import numpy as np
import pytest

from gpu_util import geom, gpu_plan, rel_l2, to_dev, to_np, tol, uniform
from oracle.gram import gram_taps
from oracle.normal import apply_direct, apply_fft, embed_size, embed_spectrum
from synth import CONFIGS
from synth.phantom import random_image

pytestmark = pytest.mark.gpu


def check_apply(bsct, g, dt, B, seed, direct=False):
    import torch
    plan, taps = gpu_plan(bsct, g, dt, max_batch=B)
    x = random_image(seed, B, g["N"])
    y = torch.empty((B, g["N"], g["N"]), dtype=taps.dtype, device="cuda")
    bsct.normal_apply(plan, to_dev(x, dt), y)
    ref_taps = gram_taps(g)
    ref = apply_direct(ref_taps, x) if direct else apply_fft(ref_taps, x)
    for i in range(B):
        assert rel_l2(to_np(y[i]), ref[i]) < tol(dt), i
    return plan, taps


@pytest.mark.parametrize("N,n,zeta,dt,B", [
    (1, 4, 0.0, "f32", 2), (2, 5, 1.0, "f32", 3), (3, 6, 0.5, "f64", 2), (5, 9, 1.0, "f32", 3),
    (8, 12, 0.0, "f32", 1), (13, 20, 1.0, "f64", 2), (24, 30, 1.0, "f32", 2), (37, 40, 0.5, "f32", 3),
    (100, 60, 1.0, "f32", 2), (129, 64, 1.0, "f32", 1), (200, 50, 1.0, "f32", 2), (256, 45, 0.0, "f32", 3), (257, 30, 0.5, "f32", 2), (300, 40, 1.0, "f32", 1), (701, 24, 1.0, "f32", 2)])
def test_small_and_ragged(cuda_lib, N, n, zeta, dt, B):
    check_apply(cuda_lib, geom(N, uniform(n), 2 * N + 1, zeta=zeta), dt, B, seed=N, direct=N <= 24)


@pytest.mark.parametrize("ci,B", [(1, 3), (2, 2), (3, 2), (4, 1)])
def test_configs(cuda_lib, ci, B):
    cfg = CONFIGS[ci]
    check_apply(cuda_lib, cfg.geometry(), cfg.dtype, B, seed=100 + ci)


def test_spectrum(cuda_lib):
    import torch
    for N, dt in ((5, "f32"), (64, "f64"), (256, "f32")):
        g = geom(N, uniform(45), 2 * N + 1, zeta=1.0)
        plan, taps = gpu_plan(cuda_lib, g, dt)
        L = embed_size(N)
        assert plan.L == L
        S = torch.empty((L // 2 + 1, L), dtype=taps.dtype, device="cuda")
        cuda_lib.plan_spectrum(plan, S)
        ref = embed_spectrum(gram_taps(g)) / (L * L)       # [p][q]
        assert rel_l2(to_np(S), ref[:, :L // 2 + 1].T) < tol(dt)


def test_delta_and_inplace(cuda_lib):
    import torch
    N = 31
    g = geom(N, uniform(30), 63, zeta=1.0)
    plan, taps = gpu_plan(cuda_lib, g, "f32", max_batch=2)
    x = torch.zeros((1, N, N), device="cuda")
    x[0, N // 2, N // 2] = 1.0
    cuda_lib.normal_apply(plan, x, x)                        # x == y allowed
    c = N - 1 - N // 2
    ref = to_np(taps)[c:c + N, c:c + N]
    assert rel_l2(to_np(x[0]), ref) < 1e-6
    cuda_lib.normal_apply(plan, x[:0], x[:0])                # B = 0: no-op
    with pytest.raises(cuda_lib.BsctError):
        cuda_lib.normal_apply(plan, torch.zeros((3, N, N), device="cuda"), torch.zeros((3, N, N), device="cuda"))


def test_psd_on_device(cuda_lib):
    """<x, Gx> >= 0 for random x through the CUDA path (G = H^T H)."""
    import torch
    g = CONFIGS[2].geometry()
    plan, taps = gpu_plan(cuda_lib, g, "f32", max_batch=4)
    x = to_dev(random_image(7, 4, g["N"]), "f32")
    y = torch.empty_like(x)
    cuda_lib.normal_apply(plan, x, y)
    assert ((x.double() * y.double()).sum(dim=(1, 2)) > 0).all()
