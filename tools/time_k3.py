"""K3 + K4 device times at config 5 (library events around every launch): python tools/time_k3.py [B]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_13471_b200 as bsct  # noqa: E402
from synth import CONFIGS  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
cfg = CONFIGS[5]
g = cfg.geometry()
N = g["N"]
taps = torch.empty((2 * N - 1, 2 * N - 1), dtype=torch.float32, device="cuda")
bsct.gram_build(g, taps)
plan = bsct.plan_create(g, taps, max_batch=B)
sino = torch.rand((B, len(g["angles"]), g["n_det"]), device="cuda")
b = torch.empty((B, N, N), device="cuda")
for _ in range(2):
    bsct.backproject(plan, sino, b)
torch.cuda.synchronize()
plan.profile(True)
for _ in range(5):
    bsct.backproject(plan, sino, b)
torch.cuda.synchronize()
pr = plan.profile_read()
print(os.environ.get("BSCT_LIB", "default"), {k: round(v[0] / 5, 3) for k, v in pr.items()}, flush=True)
