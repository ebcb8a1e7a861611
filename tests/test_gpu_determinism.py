"""R20: every kernel reduces in a fixed order (no float atomics), so repeated
runs are bitwise identical -- Gram build, back projection, every solver path, SIRT, Chebyshev."""
import numpy as np
import pytest

from gpu_util import gpu_plan, to_dev
from synth import CONFIGS
from synth.sinogram import random_sinogram

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ci,onchip", [(2, "0"), (2, "1"), (3, "0")])
def test_repeat_bitwise(cuda_lib, ci, onchip, monkeypatch):
    import torch
    monkeypatch.setenv("BSCT_ONCHIP", onchip)
    cfg = CONFIGS[ci].with_(n_angles=60, n_det=2 * CONFIGS[ci].N + 3)
    g = cfg.geometry()
    N, B = cfg.N, 3
    sino = to_dev(np.abs(random_sinogram(7, B, cfg.n_angles, cfg.n_det)), "f32")
    outs = []
    for _ in range(2):
        plan, taps = gpu_plan(cuda_lib, g, "f32", max_batch=B)
        res = [taps.clone()]
        for solver in ("cg", "sd", "landweber"):
            x = torch.empty((B, N, N), device="cuda")
            cuda_lib.reconstruct(plan, sino, x, 6, solver)
            res.append(x)
        b = torch.empty((B, N, N), device="cuda")
        cuda_lib.backproject(plan, sino, b)
        xc = torch.empty_like(b)
        cuda_lib.chebyshev_solve(plan, b, xc, 6, 1e-3)
        xs = torch.empty_like(b)
        cuda_lib.sirt_solve(plan, sino, xs, 3)
        res += [b, xc, xs]
        torch.cuda.synchronize()
        outs.append([r.cpu() for r in res])
    for a, c in zip(*outs):
        assert torch.equal(a, c)
