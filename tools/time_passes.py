"""A/B timing of the warp-FFT passes against the generic block-FFT passes at one config's
geometry: python tools/time_passes.py CONFIG BATCH ITERS (toggles BSCT_PASSB_V1/BSCT_PASSC_V1
per run; the library reads them per call)."""
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
dt = torch.float64 if cfg.dtype == "f64" else torch.float32
taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda", dtype=dt)
bsct.gram_build(g, taps)
plan = bsct.plan_create(g, taps, max_batch=B)
b = torch.rand((B, N, N), device="cuda", dtype=dt)
x = torch.empty_like(b)
for name, env in (("warp", {}), ("generic B", {"BSCT_PASSB_V1": "1"}),
                  ("generic B+C", {"BSCT_PASSB_V1": "1", "BSCT_PASSC_V1": "1"}), ("warp again", {})):
    for k in ("BSCT_PASSB_V1", "BSCT_PASSC_V1"):
        os.environ.pop(k, None)
    os.environ.update(env)
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
    ms = min(ts)
    plan.profile(True)
    bsct.cg_solve(plan, b, x, K, "cg")
    prof = {k: round(v[0], 2) for k, v in plan.profile_read().items() if v[0] > 0.05}
    plan.profile(False)
    print(f"config {ci} N={N} L={plan.L} B={B} K={K} {name:12s}: {ms:8.2f} ms  "
          f"{B * K / ms * 1e3:10.0f} slice-iter/s  {ms / K * 1e3 / B:7.2f} us/slice-iter  {prof}", flush=True)
