"""Small-problem solve timing (configs 2 and 1): fused 3-launch iteration with / without CUDA-graph
replay, and the NEXT-2 cluster-resident loop (onchip.cu)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2005_13471_b200 as bsct
from synth import CONFIGS

out = []
for ci, Bs in ((2, (1, 16, 128)), (1, (1, 64))):
    cfg = CONFIGS[ci]
    g = cfg.geometry()
    N = cfg.N
    dt = torch.float64 if cfg.dtype == "f64" else torch.float32
    taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda", dtype=dt)
    bsct.gram_build(g, taps)
    for B in Bs:
        plan = bsct.plan_create(g, taps, max_batch=B)
        b = torch.rand((B, N, N), device="cuda", dtype=dt)
        x = torch.empty_like(b)
        row = {"config": ci, "N": N, "B": B, "iters": cfg.iters, "dtype": cfg.dtype}
        for mode, onchip, graph in (("onchip_ms", "1", "1"), ("fused_ms", "0", "1"), ("fused_nograph_ms", "0", "0")):
            os.environ["BSCT_ONCHIP"] = onchip
            os.environ["BSCT_GRAPH"] = graph
            bsct.cg_solve(plan, b, x, cfg.iters, "cg")
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                bsct.cg_solve(plan, b, x, cfg.iters, "cg")
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            row[mode] = ms
        row["graph_speedup"] = row["fused_nograph_ms"] / row["fused_ms"]
        row["onchip_slice_iter_s"] = B * cfg.iters / (row["onchip_ms"] / 1e3)
        out.append(row)
        print(json.dumps(row), flush=True)
