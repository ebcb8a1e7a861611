"""Pass B probe: one CG solve on B slices of a config's geometry, per-kernel-class times (library
profiler).  python tools/pb_probe.py CONFIG B ITERS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2005_13471_b200 as bsct
from synth import CONFIGS

ci, B, K = (int(a) for a in sys.argv[1:4])
cfg = CONFIGS[ci]
g = cfg.geometry()
N = cfg.N
taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
bsct.gram_build(g, taps)
plan = bsct.plan_create(g, taps, max_batch=B)
b = torch.rand((B, N, N), device="cuda")
x = torch.empty_like(b)
bsct.cg_solve(plan, b, x, K, "cg")
torch.cuda.synchronize()
plan.profile(True)
bsct.cg_solve(plan, b, x, K, "cg")
prof = plan.profile_read()
print({k: round(v[0] / v[1], 4) for k, v in prof.items()})
