"""One config-5 CG solve of B slices x K iterations with the current BSCT_* env (for ncu probes of
the L2-resident chunk mode): python tools/l2_probe.py B K"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2005_13471_b200 as bsct
from synth import CONFIGS

B, K = int(sys.argv[1]), int(sys.argv[2])
cfg = CONFIGS[5]
g = cfg.geometry()
N = cfg.N
taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
bsct.gram_build(g, taps)
plan = bsct.plan_create(g, taps, max_batch=B)
b = torch.rand((B, N, N), device="cuda")
x = torch.empty_like(b)
for _ in range(2):
    bsct.cg_solve(plan, b, x, K, "cg")
torch.cuda.synchronize()
print("ok")
