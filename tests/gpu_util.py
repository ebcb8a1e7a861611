"""Helpers for the GPU parity tests (CUDA path vs the FP64 oracle)."""
from __future__ import annotations

import numpy as np


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def tol(dtype: str) -> float:
    """north_star: 1e-5 relative L2 for FP32 filters / single operator applications;
    SURVEY.md R19 for FP64: 1e-10."""
    return 1e-10 if dtype == "f64" else 1e-5


def torch_dtype(dtype: str):
    import torch
    return torch.float64 if dtype == "f64" else torch.float32


def to_dev(a, dtype: str):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch_dtype(dtype), device="cuda")


def to_np(t):
    return t.detach().double().cpu().numpy()


def geom(N, angles, n_det, lambda_y=1.0, zeta=0.0, lambda_x=1.0):
    return dict(N=N, lambda_x=lambda_x, angles=np.asarray(angles, dtype=np.float64), lambda_y=lambda_y,
                n_det=n_det, zeta=zeta)


def uniform(n):
    return np.arange(n) * np.pi / n


def gpu_taps(bsct, g, dtype):
    import torch
    N = g["N"]
    taps = torch.empty((2 * N - 1, 2 * N - 1), dtype=torch_dtype(dtype), device="cuda")
    bsct.gram_build(g, taps)
    return taps


def gpu_plan(bsct, g, dtype, max_batch=1):
    taps = gpu_taps(bsct, g, dtype)
    return bsct.plan_create(g, taps, max_batch=max_batch), taps
