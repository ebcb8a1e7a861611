"""L2-resident solver chunks at L = 2048 (config 4 geometry, B = 16 and 32): BSCT_CG_CHUNK x
BSCT_CHUNK_STREAMS against the whole-batch launches, CUDA-event time of bsct_cg_solve, us per
slice-iteration (20 iterations)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2005_13471_b200 as bsct
from synth import CONFIGS

ci = int(os.environ.get("CONFIG", "4"))
cfg = CONFIGS[ci]
g = cfg.geometry()
N, K = cfg.N, 20
taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
bsct.gram_build(g, taps)
for B in [int(v) for v in os.environ.get("BATCHES", "16,32").split(",")]:
    plan = bsct.plan_create(g, taps, max_batch=B)
    b = torch.rand((B, N, N), device="cuda")
    x = torch.empty_like(b)
    ref = None
    for chunk, streams in (("0", "1"), ("1", "2"), ("1", "4"), ("2", "2"), ("2", "4"), ("4", "2"), ("4", "4"), ("1", "8")):
        os.environ["BSCT_CG_CHUNK"] = chunk
        os.environ["BSCT_CHUNK_STREAMS"] = streams
        for _ in range(2):
            bsct.cg_solve(plan, b, x, K, "cg")
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            bsct.cg_solve(plan, b, x, K, "cg")
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        if ref is None:
            ref = x.clone()
        same = bool(torch.equal(ref, x))
        ms = sorted(ts)[2]
        print(json.dumps({"config": ci, "N": N, "B": B, "chunk": chunk, "streams": streams, "ms": round(ms, 3),
                          "us_per_slice_iter": round(1e3 * ms / (B * K), 2), "bitwise_equal_whole_batch": same}),
              flush=True)
    del plan
