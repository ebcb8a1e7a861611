"""Solver parity at the large configs and R12 check (ii).

* SD and Landweber at configs 4 and 5 at the configured iteration count, 1e-3 (north_star:
  "1e-3 on reconstructions after the configured iteration count"); config 5 on B = 4 slices of
  its geometry (distinct phantoms).
* FP32 CG at configs 4 and 5: x_k within 1e-4 for k <= 5 and the objective guard
  f(x_K) <= f(x_oracle at ceil(0.8 K)) (R12 (i), (iii)).  Config 4 (N = 1024, lambda_y = 0.5,
  zeta = 0.5) runs the fused CG-mode L = 2048 passes with N = L/2.
* R12 (ii): one CG step on the GPU from the oracle's own state (x, r, p) after K-1 iterations
  (bsct_cg_resume): x_K and alpha_{K-1} within 1e-5 of the oracle's, at configs 1-5.
* bsct_cg_resume: resuming from (0, b, b) is bitwise the plain solve; a solve split in two
  resumed pieces matches the unsplit one.
"""
import functools

import numpy as np
import pytest

from gpu_util import gpu_plan, rel_l2, to_dev, to_np
from oracle import solvers
from oracle.gram import gram_taps
from oracle.normal import apply_fft
from synth import CONFIGS
from synth.phantom import config_image

pytestmark = pytest.mark.gpu


@functools.lru_cache(maxsize=None)
def oracle_taps(ci):
    return gram_taps(CONFIGS[ci].geometry())


@functools.lru_cache(maxsize=None)
def rhs(ci, B=1):
    T = oracle_taps(ci)
    return np.stack([apply_fft(T, config_image(CONFIGS[ci], s)) for s in range(B)])


@functools.lru_cache(maxsize=None)
def plan_for(bsct_id, ci, B):
    import paper_2005_13471_b200 as bsct
    cfg = CONFIGS[ci]
    return gpu_plan(bsct, cfg.geometry(), cfg.dtype, max_batch=B)


def run(bsct, ci, b, iters, solver):
    import torch
    cfg = CONFIGS[ci]
    B = b.shape[0]
    plan, taps = plan_for(id(bsct), ci, max(B, 4))
    x = torch.empty((B, cfg.N, cfg.N), dtype=taps.dtype, device="cuda")
    hist = torch.empty((B, max(iters, 1)), dtype=torch.float64, device="cuda")
    flags = torch.empty((B,), dtype=torch.int32, device="cuda")
    bsct.cg_solve(plan, to_dev(b, cfg.dtype), x, iters, solver, resid_hist=hist, flags=flags)
    torch.cuda.synchronize()
    assert not flags.any()
    return to_np(x), hist.cpu().numpy()


@pytest.mark.parametrize("ci,B", [(4, 1), (5, 4)])
@pytest.mark.parametrize("solver", ["sd", "landweber"])
def test_sd_landweber_large(cuda_lib, ci, B, solver):
    cfg = CONFIGS[ci]
    T = oracle_taps(ci)
    b = rhs(ci, B)
    x, h = run(cuda_lib, ci, b, cfg.iters, solver)
    f = solvers.sd if solver == "sd" else solvers.landweber
    for s in range(B):
        xr, hr = f(T, b[s], cfg.iters)
        assert rel_l2(x[s], xr) < 1e-3
        assert rel_l2(h[s], hr) < 1e-3


@pytest.mark.parametrize("ci", [4, 5])
def test_cg_fp32_large(cuda_lib, ci):
    cfg = CONFIGS[ci]
    T = oracle_taps(ci)
    b = rhs(ci)
    x5, _ = run(cuda_lib, ci, b, 5, "cg")
    xr5, _ = solvers.cg(T, b[0], 5)
    assert rel_l2(x5[0], xr5) < 1e-4
    K = cfg.iters
    x, _ = run(cuda_lib, ci, b, K, "cg")
    xk, _ = solvers.cg(T, b[0], int(np.ceil(0.8 * K)))
    assert solvers.objective(T, b[0], x[0]) <= solvers.objective(T, b[0], xk)


def resume(bsct, ci, x, r, p, iters, solver="cg"):
    import torch
    cfg = CONFIGS[ci]
    B = x.shape[0]
    plan, taps = plan_for(id(bsct), ci, max(B, 4))
    xd, rd = to_dev(x, cfg.dtype), to_dev(r, cfg.dtype)
    pd = to_dev(p, cfg.dtype) if p is not None else None
    alpha = torch.empty((B,), dtype=torch.float64, device="cuda")
    hist = torch.empty((B, max(iters, 1)), dtype=torch.float64, device="cuda")
    bsct.cg_resume(plan, xd, rd, pd, iters, solver, alpha_last=alpha, resid_hist=hist)
    torch.cuda.synchronize()
    return xd, rd, pd, alpha.cpu().numpy(), hist.cpu().numpy()


@pytest.mark.parametrize("ci", [1, 2, 3, 4, 5])
def test_cg_one_step_from_oracle_state(cuda_lib, ci):
    """R12 (ii): start from the oracle's state after K-1 iterations, take one GPU CG step."""
    cfg = CONFIGS[ci]
    T = oracle_taps(ci)
    b = rhs(ci)[0]
    K = cfg.iters
    rec = []
    solvers.cg(T, b, K, record=rec)
    s = rec[K - 2]  # state after iteration K-1 (x_{K-1}, r_{K-1}, p_{K-1})
    xd, rd, pd, alpha, _ = resume(cuda_lib, ci, s["x"][None], s["r"][None], s["p"][None], 1)
    tl = 1e-10 if cfg.dtype == "f64" else 1e-5
    assert abs(alpha[0] - rec[K - 1]["alpha"]) <= tl * abs(rec[K - 1]["alpha"])
    assert rel_l2(to_np(xd)[0], rec[K - 1]["x"]) < tl
    assert rel_l2(to_np(rd)[0], rec[K - 1]["r"]) < (1e-8 if cfg.dtype == "f64" else 1e-3)


@pytest.mark.parametrize("ci", [1, 2, 5])
@pytest.mark.parametrize("solver", ["cg", "sd", "landweber"])
def test_resume_from_start_is_the_solve(cuda_lib, ci, solver):
    """(x, r, p) = (0, b, b) resumed for K iterations is bitwise the plain solve."""
    import torch
    cfg = CONFIGS[ci]
    B = 2
    b = rhs(ci, B)
    K = 7
    xs, hs = run(cuda_lib, ci, b, K, solver)
    xd, rd, pd, _, hr = resume(cuda_lib, ci, np.zeros_like(b), b, b if solver == "cg" else None, K, solver)
    assert np.array_equal(to_np(xd), xs)
    assert np.array_equal(hr, hs)


@pytest.mark.parametrize("ci", [1, 2, 4])
def test_resume_split_solve(cuda_lib, ci):
    """A CG solve split into two resumed pieces (the exported state of the first feeds the second)
    matches the unsplit solve; the exported r is the oracle's r_j."""
    cfg = CONFIGS[ci]
    b = rhs(ci)
    K, j = 8, 3
    xs, _ = run(cuda_lib, ci, b, K, "cg")
    xd, rd, pd, _, _ = resume(cuda_lib, ci, np.zeros_like(b), b, b, j)
    x1, r1, p1 = to_np(xd), to_np(rd), to_np(pd)
    rec = []
    solvers.cg(oracle_taps(ci), b[0], j, record=rec)
    tl = 1e-10 if cfg.dtype == "f64" else 1e-4
    assert rel_l2(r1[0], rec[-1]["r"]) < tl
    assert rel_l2(p1[0], rec[-1]["p"]) < tl
    xd2, _, _, _, _ = resume(cuda_lib, ci, x1, r1, p1, K - j)
    assert rel_l2(to_np(xd2), xs) < (1e-12 if cfg.dtype == "f64" else 1e-5)
