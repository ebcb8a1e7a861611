"""Desk-scale reconstruction-quality harness.

The paper's experiments (detector downsampling n = lambda_y / lambda_x in
[0.25, 2], blurred vs unblurred detector model, SNR / SSIM on "Spots" / Forbild / LIDC)
need images and baselines that are not available here; this harness runs the same kind
of sweep on seeded synthetic phantoms through the library only:

* phantom: 30 random ellipses (config-2 recipe, N = 256), reference image = its 4x4
  supersampled pixel-coefficient rasterisation (synth.phantom);
* data: analytic line integrals averaged over detector cells of width lambda_y (a true
  box detector) at 180 views, n_det covering the field of view, optional
  Gaussian noise (sigma = level x max);
* model: the paper's box-spline pixel model with detector blur zeta_model = lambda_y
  ("blurred", Eq.(4)) or zeta_model = 0 (Eq.(3), blur not modelled);
* solvers: steepest descent (the paper's) and CG on G x = H^T g^;
* metrics ("SNR and SSIM"): SNR = 10 log10(||f||^2 / ||f - x||^2) against the reference
  image, and the mean structural similarity SSIM (Wang et al. 2004; the constants of SPEC S:407-410:
  11 x 11 Gaussian window sigma = 1.5, K1 = 0.01, K2 = 0.03, dynamic range L = max - min of the
  reference; windows inside the image only).

    python tools/experiments.py [--N 256] [--iters 50] [--out profiles/r01/experiments.md]

No baselines (sinc / oblique / orthogonal methods are out of scope); the numbers are
this implementation's, for the record.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def snr_db(ref: np.ndarray, x: np.ndarray) -> float:
    err = float(np.sum((ref - x) ** 2))
    return float("inf") if err == 0 else 10.0 * math.log10(float(np.sum(ref ** 2)) / err)


def _gauss_window(size: int = 11, sigma: float = 1.5) -> np.ndarray:
    k = np.arange(size) - (size - 1) / 2.0
    w = np.exp(-k ** 2 / (2.0 * sigma ** 2))
    return w / w.sum()


def _filter_valid(img: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Separable correlation with the 1-D window w on both axes, 'valid' region only."""
    n = w.size
    rows = sum(w[i] * img[i:img.shape[0] - n + 1 + i, :] for i in range(n))
    return sum(w[j] * rows[:, j:img.shape[1] - n + 1 + j] for j in range(n))


def ssim(ref: np.ndarray, x: np.ndarray, size: int = 11, sigma: float = 1.5, k1: float = 0.01,
         k2: float = 0.03) -> float:
    """Mean SSIM over the 'valid' windows: per window
    ((2 mu_r mu_x + C1)(2 s_rx + C2)) / ((mu_r^2 + mu_x^2 + C1)(s_r^2 + s_x^2 + C2)),
    Gaussian-weighted moments, C1 = (k1 L)^2, C2 = (k2 L)^2, L = max(ref) - min(ref)."""
    ref = np.asarray(ref, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    if ref.shape != x.shape:
        raise ValueError("size mismatch")
    if min(ref.shape) < size:
        raise ValueError(f"images must be at least {size} x {size}")
    L = float(ref.max() - ref.min())
    if L == 0:
        raise ValueError("constant reference")
    c1, c2 = (k1 * L) ** 2, (k2 * L) ** 2
    w = _gauss_window(size, sigma)
    mr, mx = _filter_valid(ref, w), _filter_valid(x, w)
    srr = _filter_valid(ref * ref, w) - mr * mr
    sxx = _filter_valid(x * x, w) - mx * mx
    srx = _filter_valid(ref * x, w) - mr * mx
    m = ((2 * mr * mx + c1) * (2 * srx + c2)) / ((mr * mr + mx * mx + c1) * (srr + sxx + c2))
    return float(m.mean())


def problem(N, n_views, ratio, noise, seed):
    """Reference image, sinogram and base geometry of one sweep point (no library call)."""
    from synth.phantom import random_ellipses, rasterize_ellipses
    from synth.sinogram import add_gaussian_noise, ellipse_sinogram
    ell = random_ellipses(seed, 30, N / 64.0)
    ref = rasterize_ellipses(ell, N, 1.0)
    angles = np.arange(n_views) * np.pi / n_views
    ly = float(ratio)
    n_det = int(math.ceil(N * math.sqrt(2.0) / ly)) | 1
    sino = ellipse_sinogram(ell, angles, n_det, ly, ly)  # box detector of width lambda_y
    if noise:
        sino = add_gaussian_noise(sino, seed + 1, noise)
    return ref, sino, dict(N=N, lambda_x=1.0, angles=angles, lambda_y=ly, n_det=n_det)


def reconstruct_gpu(g, sino, solvers, iters):
    """x = solver^iters(G, H^T g^) through the library, one reconstruction per solver."""
    import torch

    import paper_2005_13471_b200 as bsct
    N = g["N"]
    taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
    bsct.gram_build(g, taps)
    plan = bsct.plan_create(g, taps, max_batch=1)
    s = torch.as_tensor(sino[None], dtype=torch.float32, device="cuda")
    b = torch.empty((1, N, N), device="cuda")
    bsct.backproject(plan, s, b)
    out = {}
    for sv in solvers:
        x = torch.empty_like(b)
        bsct.cg_solve(plan, b, x, iters, sv)
        torch.cuda.synchronize()
        out[sv] = x[0].double().cpu().numpy()
    return out


def run(N=256, n_views=180, ratios=(0.25, 0.5, 1.0, 2.0), noise=(0.0, 0.005), iters=50, seed=2000,
        solvers=("sd", "cg")):
    import paper_2005_13471_b200 as bsct
    bsct.load()
    rows = []
    for n in ratios:
        for lvl in noise:
            ref, sino, g0 = problem(N, n_views, n, lvl, seed)
            for zeta in (float(n), 0.0):
                xs = reconstruct_gpu(dict(g0, zeta=zeta), sino, solvers, iters)
                for sv in solvers:
                    rows.append(dict(ratio=n, noise=lvl, model="blurred" if zeta > 0 else "unblurred",
                                     solver=sv, iters=iters, snr_db=snr_db(ref, xs[sv]), ssim=ssim(ref, xs[sv])))
    return rows


def to_markdown(rows, N, iters) -> str:
    out = [f"# Reconstruction quality sweep (tools/experiments.py; N = {N}, 180 views, {iters} iterations)",
           "",
           "SNR (dB) / SSIM against the 4x4-supersampled pixel image of a 30-ellipse phantom; data = exact",
           "line integrals averaged over box detector cells of width lambda_y (+ Gaussian noise);",
           "model blur zeta = lambda_y (blurred, Eq.(4)) or 0 (unblurred, Eq.(3)).  No baselines.",
           "",
           "| n = ly/lx | noise | solver | blurred model SNR / SSIM | unblurred model SNR / SSIM |",
           "|---|---|---|---|---|"]
    keys = sorted({(r["ratio"], r["noise"], r["solver"]) for r in rows})
    for (n, lvl, sv) in keys:
        val = {r["model"]: (r["snr_db"], r["ssim"]) for r in rows
               if (r["ratio"], r["noise"], r["solver"]) == (n, lvl, sv)}
        nan = (float("nan"), float("nan"))
        bl, ub = val.get("blurred", nan), val.get("unblurred", nan)
        out.append(f"| {n} | {lvl:g} | {sv} | {bl[0]:.2f} / {bl[1]:.4f} | {ub[0]:.2f} / {ub[1]:.4f} |")
    return "\n".join(out) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=256)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = run(N=a.N, iters=a.iters)
    md = to_markdown(rows, a.N, a.iters)
    print(md)
    for r in rows:
        print(json.dumps(r))
    if a.out:
        with open(a.out, "w") as f:
            f.write(md + "\n```\n" + "\n".join(json.dumps(r) for r in rows) + "\n```\n")


if __name__ == "__main__":
    main()
