"""Time K7 (forward projection) v3 vs v1 on config-5 geometry, 64 slices."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2005_13471_b200 as bsct
from synth import CONFIGS
cfg = CONFIGS[5]; g = cfg.geometry(); N = cfg.N; B = 64
taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda"); bsct.gram_build(g, taps)
plan = bsct.plan_create(g, taps, max_batch=B)
x = torch.rand((B, N, N), device="cuda")
out = {}
for v in ("1", "0"):
    os.environ["BSCT_FWD_V1"] = v
    s = torch.empty((B, cfg.n_angles, cfg.n_det), device="cuda")
    bsct.forward_project(plan, x, s); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); bsct.forward_project(plan, x, s); e1.record(); torch.cuda.synchronize()
    out["v1" if v == "1" else "v3"] = (e0.elapsed_time(e1), s.clone())
d = float((out["v1"][1] - out["v3"][1]).norm() / out["v1"][1].norm())
print(json.dumps({"v1_ms": out["v1"][0], "v3_ms": out["v3"][0], "rel_diff": d,
                  "v3_gvox_angle_s": B * N * N * cfg.n_angles / (out["v3"][0] / 1e3) / 1e9}))
