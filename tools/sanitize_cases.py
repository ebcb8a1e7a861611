"""Small invocations of every kernel family with shared-memory staging or block/cluster
synchronisation, for compute-sanitizer (racecheck / synccheck / memcheck, one tool per run):

  K0 tables, K1 Gram tiles (levels 0-2, dense mode), K2 spectrum, K3 correction, K4 v3 back
  projection (cp.async ring), K5 warp-FFT passes A/B/C at L = 512, 1024, 2048 (fused CG, SD,
  plain apply), generic passes (other L, FP64), K7 forward, NEXT-2 on-chip cluster solver (DSMEM),
  CG resume.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2005_13471_b200 as bsct
    bsct.load()
    dev = torch.device("cuda")
    gen = torch.Generator(device=dev).manual_seed(0)
    cases = [(257, 40, "f32"), (513, 24, "f32"), (1025, 16, "f32"), (100, 30, "f32"), (40, 30, "f64")]
    for N, n, dt in cases:
        tdt = torch.float64 if dt == "f64" else torch.float32
        M = int(1.5 * N) | 1
        g = dict(N=N, lambda_x=1.0, angles=np.arange(n) * np.pi / n + 0.01, lambda_y=1.0, n_det=M, zeta=1.0)
        taps = torch.empty((2 * N - 1, 2 * N - 1), dtype=tdt, device=dev)
        bsct.gram_build(g, taps)
        os.environ["BSCT_GRAM_DENSE"] = "1"
        bsct.gram_build(g, taps)
        del os.environ["BSCT_GRAM_DENSE"]
        B = 2
        plan = bsct.plan_create(g, taps, max_batch=B)
        sino = torch.rand((B, n, M), dtype=tdt, device=dev, generator=gen)
        b = torch.empty((B, N, N), dtype=tdt, device=dev)
        bsct.backproject(plan, sino, b)
        x = torch.empty_like(b)
        for sv in ("cg", "sd", "landweber"):
            bsct.cg_solve(plan, b, x, 2, sv)
        y = torch.empty_like(b)
        bsct.normal_apply(plan, x, y)
        bsct.forward_project(plan, x, sino)
        r = b.clone()
        p = b.clone()
        bsct.cg_resume(plan, torch.zeros_like(b), r, p, 2)
        torch.cuda.synchronize()
        print(f"N={N} n={n} {dt}: ok", flush=True)
    # NEXT-2 on-chip cluster solver (DSMEM), N <= 256
    os.environ["BSCT_ONCHIP"] = "1"
    for N, dt in ((64, "f64"), (200, "f32"), (256, "f32")):
        tdt = torch.float64 if dt == "f64" else torch.float32
        g = dict(N=N, lambda_x=1.0, angles=np.arange(24) * np.pi / 24, lambda_y=1.0, n_det=2 * N + 1, zeta=1.0)
        taps = torch.empty((2 * N - 1, 2 * N - 1), dtype=tdt, device=dev)
        bsct.gram_build(g, taps)
        plan = bsct.plan_create(g, taps, max_batch=2)
        b = torch.rand((2, N, N), dtype=tdt, device=dev, generator=gen)
        x = torch.empty_like(b)
        for sv in ("cg", "sd", "landweber"):
            bsct.cg_solve(plan, b, x, 2, sv)
        torch.cuda.synchronize()
        print(f"onchip N={N} {dt}: ok", flush=True)
    del os.environ["BSCT_ONCHIP"]


if __name__ == "__main__":
    main()
