"""GPU parity for NEXT-1: plain adjoint H^T and SIRT vs oracle.forward.adjoint
and oracle.sirt (FP32 1e-5 / FP64 1e-10 relative L2 for the operator; SIRT is linear in the
data, so its iterates keep FP32 parity: 1e-4 after the configured iterations)."""
import numpy as np
import pytest

from gpu_util import geom, gpu_plan, rel_l2, to_dev, to_np, tol, uniform
from oracle.forward import adjoint
from oracle.sirt import sirt
from synth import CONFIGS
from synth.sinogram import random_sinogram

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,n,M,ly,zeta,dt,B", [
    (5, 7, 13, 1.0, 0.0, "f32", 1), (8, 12, 19, 0.8, 1.0, "f64", 2), (16, 20, 33, 1.0, 1.5, "f32", 5),
    (33, 30, 49, 0.5, 0.5, "f32", 2), (12, 9, 25, 1.3, 0.7, "f64", 1)])
def test_adjoint_small(cuda_lib, N, n, M, ly, zeta, dt, B):
    import torch
    g = geom(N, uniform(n) + 0.013, M, lambda_y=ly, zeta=zeta)
    sino = random_sinogram(N + 7, B, n, M)
    plan, taps = gpu_plan(cuda_lib, g, dt, max_batch=B)
    out = torch.empty((B, N, N), dtype=taps.dtype, device="cuda")
    cuda_lib.adjoint_project(plan, to_dev(sino, dt), out)
    for i in range(B):
        assert rel_l2(to_np(out[i]), adjoint(g, sino[i])) < tol(dt)


def test_adjoint_dot_product_on_device(cuda_lib):
    """<H c, g> = <c, H^T g> through the CUDA forward and adjoint (config-2 geometry)."""
    import torch
    g = CONFIGS[2].geometry()
    N = g["N"]
    plan, taps = gpu_plan(cuda_lib, g, "f32", max_batch=1)
    rng = np.random.default_rng(9)
    c = to_dev(rng.uniform(-1, 1, (1, N, N)), "f32")
    s = to_dev(rng.uniform(-1, 1, (1, len(g["angles"]), g["n_det"])), "f32")
    hc = torch.empty_like(s)
    cuda_lib.forward_project(plan, c, hc)
    hts = torch.empty_like(c)
    cuda_lib.adjoint_project(plan, s, hts)
    lhs = float((hc.double() * s.double()).sum())
    rhs = float((c.double() * hts.double()).sum())
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs)


@pytest.mark.parametrize("N,n,M,zeta,dt,iters", [(8, 10, 17, 1.0, "f64", 6), (16, 24, 35, 0.5, "f32", 10),
                                                  (24, 30, 49, 1.5, "f32", 8)])
def test_sirt(cuda_lib, N, n, M, zeta, dt, iters):
    import torch
    g = geom(N, uniform(n) + 0.05, M, zeta=zeta)
    sino = np.abs(random_sinogram(3 * N, 2, n, M))
    plan, taps = gpu_plan(cuda_lib, g, dt, max_batch=2)
    x = torch.empty((2, N, N), dtype=taps.dtype, device="cuda")
    cuda_lib.sirt_solve(plan, to_dev(sino, dt), x, iters)
    for i in range(2):
        xr, _ = sirt(g, sino[i], iters)
        assert rel_l2(to_np(x[i]), xr) < (1e-10 if dt == "f64" else 1e-4)


def test_adjoint_config_sampled(cuda_lib):
    """Full config-5 geometry, 4 slices (K4 v3 launch with 4 slices per CTA), sampled pixels."""
    import torch
    cfg = CONFIGS[5]
    g = cfg.geometry()
    N = cfg.N
    sino = random_sinogram(55, 4, cfg.n_angles, cfg.n_det)
    plan, taps = gpu_plan(cuda_lib, g, "f32", max_batch=4)
    out = torch.empty((4, N, N), device="cuda")
    cuda_lib.adjoint_project(plan, to_dev(sino, "f32"), out)
    rng = np.random.default_rng(3)
    k1, k2 = rng.integers(0, N, 60), rng.integers(0, N, 60)
    for i in (0, 3):
        ref = adjoint(g, sino[i], pixels=(k1, k2))
        assert rel_l2(to_np(out[i])[k1, k2], ref) < 1e-5
