"""Hashes of the K3 (correction filter) outputs and of the K4 v4 back projection fed by them, for a
bitwise A/B of two library builds: BSCT_LIB=<other.so> python tools/k3_hash.py (same lines = equal)."""
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2005_13471_b200 as bsct  # noqa: E402
from gpu_util import geom, gpu_plan, to_dev, uniform  # noqa: E402
from synth.sinogram import random_sinogram  # noqa: E402

H = 25
for (N, n, M, ly, zeta, dt, B) in [(6, 12, 37, 1.0, 1.0, "f32", 2), (6, 12, 37, 0.7, 1.3, "f64", 3),
                                    (512, 360, 725, 1.0, 1.0, "f32", 11), (64, 40, 91, 1.0, 1.0, "f64", 9),
                                    (256, 90, 363, 1.0, 1.0, "f32", 8), (33, 36, 49, 1.0, 1.5, "f32", 2)]:
    g = geom(N, uniform(n), M, lambda_y=ly, zeta=zeta)
    sino = random_sinogram(N + n, B, n, M)
    plan, _ = gpu_plan(bsct, g, dt, max_batch=B)
    gt = torch.zeros((B, n, M + 2 * H), dtype=plan.dtype, device="cuda")
    bsct.correction_filter(plan, to_dev(sino, dt), gt)
    b = torch.zeros((B, N, N), dtype=plan.dtype, device="cuda")
    bsct.backproject(plan, to_dev(sino, dt), b)
    torch.cuda.synchronize()
    print(N, n, M, dt, B, hashlib.sha256(gt.cpu().numpy().tobytes()).hexdigest()[:16],
          hashlib.sha256(b.cpu().numpy().tobytes()).hexdigest()[:16], flush=True)
