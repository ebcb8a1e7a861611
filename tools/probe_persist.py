"""Diagnosis of the persistent L = 2048 CG at B = 1 (config 4): per-pass kernel times of the
per-pass launches (library events, plain launches), and the persistent kernel with the tiles of
some passes skipped (BSCT_PERSIST_SKIP; timing only), us per iteration."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2005_13471_b200 as bsct
from synth import CONFIGS

cfg = CONFIGS[4]
g = cfg.geometry()
N, K = cfg.N, 100
taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
bsct.gram_build(g, taps)
B = int(os.environ.get("B", "1"))
plan = bsct.plan_create(g, taps, max_batch=B)
b = torch.rand((B, N, N), device="cuda")
x = torch.empty_like(b)


def timed():
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
    return round(1e3 * sorted(ts)[2] / K, 2)


os.environ["BSCT_PERSIST"] = "0"
plan.profile(True)
bsct.cg_solve(plan, b, x, K, "cg")
torch.cuda.synchronize()
plan.profile_read()
bsct.cg_solve(plan, b, x, K, "cg")
torch.cuda.synchronize()
prof = {k: round(1e3 * v[0] / K, 2) for k, v in plan.profile_read().items() if v[0] > 0.0}
plan.profile(False)
print(json.dumps({"lib": os.environ.get("BSCT_LIB", "default"), "B": B, "per_pass_profiled_us_per_iter": prof}), flush=True)
row = {"lib": os.environ.get("BSCT_LIB", "default"), "B": B, "per_pass_graph_us_per_iter": timed()}
os.environ["BSCT_PERSIST"] = "1"
for skip in (0, 1, 2, 4, 6, 5, 3, 7):
    os.environ["BSCT_PERSIST_SKIP"] = str(skip)
    row[f"persist_skip{skip}"] = timed()
os.environ.pop("BSCT_PERSIST_SKIP")
print(json.dumps(row), flush=True)
