"""Persistent single-launch CG (BSCT_PERSIST=1) vs the per-pass launches (BSCT_PERSIST=0, CUDA
graph replay) at config 4's geometry (N = 1024, L = 2048, 720 angles, 100 iterations): CUDA-event
time of bsct_cg_solve per iteration and per slice-iteration for B = 1, 2, 4, 8, 16."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2005_13471_b200 as bsct
from synth import CONFIGS

cfg = CONFIGS[4]
g = cfg.geometry()
N, K = cfg.N, cfg.iters
taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
bsct.gram_build(g, taps)
reps = int(os.environ.get("REPS", "5"))
for B in [int(v) for v in os.environ.get("BATCHES", "1,2,4,8,16").split(",")]:
    plan = bsct.plan_create(g, taps, max_batch=B)
    torch.manual_seed(B)
    b = torch.rand((B, N, N), device="cuda")
    x = torch.empty_like(b)
    row = {"config": 4, "N": N, "B": B, "iters": K}
    for persist in ("0", "1"):
        os.environ["BSCT_PERSIST"] = persist
        for _ in range(2):
            bsct.cg_solve(plan, b, x, K, "cg")
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            bsct.cg_solve(plan, b, x, K, "cg")
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        key = "persist" if persist == "1" else "per_pass"
        row[key + "_ms"] = round(ms, 3)
        row[key + "_us_per_iter"] = round(1e3 * ms / K, 2)
        row[key + "_us_per_slice_iter"] = round(1e3 * ms / (K * B), 2)
    print(json.dumps(row), flush=True)
    del plan
