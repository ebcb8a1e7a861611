"""A/B of the TMA-pipelined pass C (passes_tma.cu) against cg_pass_c_1024_kernel at config 5:
python tools/time_passc.py [B] [K].  Full CG solves (best of 3, CUDA events), plain and with
L2-resident chunks on 4 streams; x must be bitwise equal between the two pass C kernels' runs?
No: the per-slice scalar reductions differ in order, so the comparison is relative L2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2005_13471_b200 as bsct
from synth import CONFIGS

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = CONFIGS[5]
g = cfg.geometry()
N = cfg.N
taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
bsct.gram_build(g, taps)
plan = bsct.plan_create(g, taps, max_batch=B)
torch.manual_seed(0)
b = torch.rand((B, N, N), device="cuda")
x = torch.empty_like(b)
KEYS = ("BSCT_PASSC_TMA", "BSCT_CG_CHUNK", "BSCT_CHUNK_STREAMS")


def run(env):
    for k in KEYS:
        os.environ.pop(k, None)
    os.environ.update(env)
    bsct.cg_solve(plan, b, x, K, "cg")
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bsct.cg_solve(plan, b, x, K, "cg")
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), x.clone()


ref = None
for mode in ({}, {"BSCT_CG_CHUNK": "4", "BSCT_CHUNK_STREAMS": "4"}, {"BSCT_CG_CHUNK": "8", "BSCT_CHUNK_STREAMS": "2"}):
    for tma in ("0", "1"):
        for skip in ("000",):
            env = dict(mode, BSCT_PASSC_TMA=tma, BSCT_SKIP_PASS=skip)
            ms, xv = run(env)
            d = ""
            if skip == "000":
                if ref is None:
                    ref = xv
                d = f"rel_l2 vs first {float((xv - ref).norm() / ref.norm()):.2e}"
            print(f"{env}: {ms:8.2f} ms  {ms / K / B * 1e3:6.3f} us/slice-iter  {d}", flush=True)
