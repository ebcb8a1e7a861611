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
* metric: SNR = 10 log10(||f||^2 / ||f - x||^2) against the reference image.

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


def run(N=256, n_views=180, ratios=(0.25, 0.5, 1.0, 2.0), noise=(0.0, 0.005), iters=50, seed=2000,
        solvers=("sd", "cg")):
    import torch

    import paper_2005_13471_b200 as bsct
    from synth.phantom import random_ellipses, rasterize_ellipses
    from synth.sinogram import add_gaussian_noise, ellipse_sinogram

    bsct.load()
    ell = random_ellipses(seed, 30, N / 64.0)
    ref = rasterize_ellipses(ell, N, 1.0)
    angles = np.arange(n_views) * np.pi / n_views
    rows = []
    for n in ratios:
        ly = float(n)
        n_det = int(math.ceil(N * math.sqrt(2.0) / ly)) | 1
        clean = ellipse_sinogram(ell, angles, n_det, ly, ly)  # box detector of width lambda_y
        for lvl in noise:
            sino = clean if lvl == 0 else add_gaussian_noise(clean, seed + 1, lvl)
            for zeta in (ly, 0.0):
                g = dict(N=N, lambda_x=1.0, angles=angles, lambda_y=ly, n_det=n_det, zeta=zeta)
                taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
                bsct.gram_build(g, taps)
                plan = bsct.plan_create(g, taps, max_batch=1)
                s = torch.as_tensor(sino[None], dtype=torch.float32, device="cuda")
                b = torch.empty((1, N, N), device="cuda")
                bsct.backproject(plan, s, b)
                for sv in solvers:
                    x = torch.empty_like(b)
                    bsct.cg_solve(plan, b, x, iters, sv)
                    torch.cuda.synchronize()
                    rows.append(dict(ratio=n, noise=lvl, model="blurred" if zeta > 0 else "unblurred",
                                     solver=sv, iters=iters, snr_db=snr_db(ref, x[0].double().cpu().numpy())))
                del plan
    return rows


def to_markdown(rows, N, iters) -> str:
    out = [f"# Reconstruction quality sweep (tools/experiments.py; N = {N}, 180 views, {iters} iterations)",
           "",
           "SNR (dB) against the 4x4-supersampled pixel image of a 30-ellipse phantom; data = exact",
           "line integrals averaged over box detector cells of width lambda_y (+ Gaussian noise);",
           "model blur zeta = lambda_y (blurred, Eq.(4)) or 0 (unblurred, Eq.(3)).  No baselines.",
           "",
           "| n = ly/lx | noise | solver | blurred model | unblurred model |",
           "|---|---|---|---|---|"]
    keys = sorted({(r["ratio"], r["noise"], r["solver"]) for r in rows})
    for (n, lvl, sv) in keys:
        val = {r["model"]: r["snr_db"] for r in rows if (r["ratio"], r["noise"], r["solver"]) == (n, lvl, sv)}
        out.append(f"| {n} | {lvl:g} | {sv} | {val.get('blurred', float('nan')):.2f} | "
                   f"{val.get('unblurred', float('nan')):.2f} |")
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
