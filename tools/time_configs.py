"""Single-slice reconstruction time at every BASELINE.json config geometry (BP + solver), and
the same per slice for a batch of 16."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2005_13471_b200 as bsct
from synth import CONFIGS

for ci in (1, 2, 3, 4, 5):
    cfg = CONFIGS[ci]
    g = cfg.geometry()
    N = cfg.N
    dt = torch.float64 if cfg.dtype == "f64" else torch.float32
    taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda", dtype=dt)
    for B in (1, 16):
        plan = bsct.plan_create(g, taps if bsct.gram_build(g, taps) is not None else taps, max_batch=B)
        sino = torch.rand((B, cfg.n_angles, cfg.n_det), device="cuda", dtype=dt)
        x = torch.empty((B, N, N), device="cuda", dtype=dt)
        b = torch.empty_like(x)
        bsct.reconstruct(plan, sino, x, cfg.iters, "cg")
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        bsct.backproject(plan, sino, b)
        ev[1].record()
        bsct.cg_solve(plan, b, x, cfg.iters, "cg")
        ev[2].record()
        torch.cuda.synchronize()
        bp, cg = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
        print(json.dumps({"config": ci, "N": N, "B": B, "iters": cfg.iters, "dtype": cfg.dtype, "bp_ms": round(bp, 3),
                          "cg_ms": round(cg, 3), "cg_us_per_slice_iter": round(1e3 * cg / (B * cfg.iters), 2),
                          "bp_gvox_angle_s": round(B * N * N * cfg.n_angles / (bp / 1e3) / 1e9, 1)}), flush=True)
