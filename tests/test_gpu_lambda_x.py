"""Reading R3 (lambda_x != 1: widths scale by lambda_x, footprint mass lambda_x^2, taps lambda_x^4)
through every GPU operator against the oracle: back projection (K4 v1/v2/v3), plain adjoint,
normal apply (generic and L = 1024 warp passes), CG, SIRT."""
import numpy as np
import pytest

from gpu_util import geom, gpu_plan, rel_l2, to_dev, to_np, tol, uniform
from oracle import solvers
from oracle.backproject import backproject
from oracle.forward import adjoint
from oracle.gram import gram_taps
from oracle.normal import apply_direct, apply_fft
from oracle.sirt import sirt
from synth.sinogram import random_sinogram

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("lx,ly,zeta,dt", [(0.5, 1.0, 1.0, "f32"), (1.7, 1.0, 0.5, "f32"), (0.8, 0.6, 1.2, "f64"),
                                           (1.3, 2.0, 0.0, "f32")])
def test_small_all_operators(cuda_lib, lx, ly, zeta, dt):
    import torch
    N, n, B = 20, 18, 5
    M = int(np.ceil(N * lx * 1.5 / ly)) * 2 + 7
    g = geom(N, uniform(n) + 0.02, M, lambda_y=ly, zeta=zeta, lambda_x=lx)
    plan, taps = gpu_plan(cuda_lib, g, dt, max_batch=B)
    T = gram_taps(g)
    assert rel_l2(to_np(taps), T) < tol(dt)
    sino = np.abs(random_sinogram(int(lx * 100), B, n, M))
    sd = to_dev(sino, dt)
    b = torch.empty((B, N, N), dtype=taps.dtype, device="cuda")
    cuda_lib.backproject(plan, sd, b)
    adj = torch.empty_like(b)
    cuda_lib.adjoint_project(plan, sd, adj)
    y = torch.empty_like(b)
    cuda_lib.normal_apply(plan, b, y)
    x = torch.empty_like(b)
    cuda_lib.cg_solve(plan, b, x, 4, "cg")
    xs = torch.empty_like(b)
    cuda_lib.sirt_solve(plan, sd, xs, 3)
    torch.cuda.synchronize()
    for i in (0, B - 1):
        bi = to_np(b[i])
        assert rel_l2(bi, backproject(g, sino[i])) < tol(dt)
        assert rel_l2(to_np(adj[i]), adjoint(g, sino[i])) < tol(dt)
        assert rel_l2(to_np(y[i]), apply_direct(T, bi)) < tol(dt)
        assert rel_l2(to_np(x[i]), solvers.cg(T, bi, 4, direct=True)[0]) < (1e-9 if dt == "f64" else 1e-4)
        assert rel_l2(to_np(xs[i]), sirt(g, sino[i], 3)[0]) < (1e-10 if dt == "f64" else 1e-4)


def test_warp_path_lambda_x(cuda_lib):
    """N = 300 (L = 1024 warp-FFT passes, K4 v3 with 4 slices per CTA) at lambda_x = 0.7."""
    import torch
    N, n, B = 300, 30, 4
    g = geom(N, uniform(n) + 0.01, 311, lambda_y=1.0, zeta=1.0, lambda_x=0.7)
    plan, taps = gpu_plan(cuda_lib, g, "f32", max_batch=B)
    assert plan.L == 1024
    T = gram_taps(g)
    sino = np.abs(random_sinogram(70, B, n, 311))
    b = torch.empty((B, N, N), device="cuda")
    cuda_lib.backproject(plan, to_dev(sino, "f32"), b)
    rng = np.random.default_rng(7)
    k1, k2 = rng.integers(0, N, 120), rng.integers(0, N, 120)
    assert rel_l2(to_np(b[B - 1])[k1, k2], backproject(g, sino[B - 1], pixels=(k1, k2))) < 1e-5
    y = torch.empty_like(b)
    cuda_lib.normal_apply(plan, b, y)
    assert rel_l2(to_np(y[0]), apply_fft(T, to_np(b[0]))) < 1e-5


@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_irregular_angles(cuda_lib, dt):
    """Unsorted, repeated and out-of-[0, pi) angles (the Gram window search sorts them mod pi; K4
    builds per-angle tables): taps, back projection, normal apply against the oracle."""
    import torch
    rng = np.random.default_rng(11)
    ang = np.concatenate([rng.uniform(-np.pi, 2 * np.pi, 21), [0.3, 0.3, np.pi / 2, 0.0, np.pi]])
    N, M, B = 24, 45, 2
    g = geom(N, ang, M, lambda_y=1.0, zeta=0.8)
    plan, taps = gpu_plan(cuda_lib, g, dt, max_batch=B)
    T = gram_taps(g)
    assert rel_l2(to_np(taps), T) < tol(dt)
    sino = random_sinogram(3, B, len(ang), M)
    b = torch.empty((B, N, N), dtype=taps.dtype, device="cuda")
    cuda_lib.backproject(plan, to_dev(sino, dt), b)
    y = torch.empty_like(b)
    cuda_lib.normal_apply(plan, b, y)
    for i in range(B):
        assert rel_l2(to_np(b[i]), backproject(g, sino[i])) < tol(dt)
        assert rel_l2(to_np(y[i]), apply_direct(T, to_np(b[i]))) < tol(dt)
