"""Hash of a CG solve (config-5 geometry, ragged batch) for a bitwise A/B of two library builds:
BSCT_LIB=<other.so> python tools/cg_hash.py"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_13471_b200 as bsct  # noqa: E402
from synth import CONFIGS  # noqa: E402

for ci, B, K in [(5, 26, 7), (3, 2, 9)]:
    cfg = CONFIGS[ci]
    g = cfg.geometry()
    N = cfg.N
    taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
    bsct.gram_build(g, taps)
    plan = bsct.plan_create(g, taps, max_batch=B)
    torch.manual_seed(1)
    b = torch.rand((B, N, N), device="cuda")
    x = torch.empty_like(b)
    bsct.cg_solve(plan, b, x, K, "cg")
    torch.cuda.synchronize()
    print(ci, B, K, hashlib.sha256(x.cpu().numpy().tobytes()).hexdigest()[:16], flush=True)
