"""Sweep of the chunked solve (L2-resident chunks on several streams, api.cu) at config 5's
geometry: python tools/time_groups.py [BATCH] [ITERS].  Each variant sets BSCT_CG_CHUNK /
BSCT_CHUNK_STREAMS (read per call), times cg_solve with CUDA events (best of 3) and checks that x
is bitwise equal to the plain solve: slices are independent, so chunking must not change a bit."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2005_13471_b200 as bsct
from synth import CONFIGS

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = CONFIGS[5]
g = cfg.geometry()
N = cfg.N
taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
bsct.gram_build(g, taps)
plan = bsct.plan_create(g, taps, max_batch=B)
torch.manual_seed(0)
b = torch.rand((B, N, N), device="cuda")
x = torch.empty_like(b)
KEYS = ("BSCT_CG_CHUNK", "BSCT_CHUNK_STREAMS")


def run(env):
    for k in KEYS:
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in env.items()})
    bsct.cg_solve(plan, b, x, K, "cg")
    torch.cuda.synchronize()
    ts = []
    import time
    for _ in range(3):
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        bsct.cg_solve(plan, b, x, K, "cg")
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    run.host_ms = (t1 - t0) * 1e3
    return min(ts), x.clone()


ms0, x0 = run({})
print(f"B={B} K={K} plain: {ms0:8.2f} ms  {ms0 / K * 1e3 / B:6.3f} us/slice-iter", flush=True)
variants = []
SWEEP = sys.argv[3] if len(sys.argv) > 3 else "1:6,1:8,2:5,2:6,2:8,3:4,3:5,3:6,4:3,4:4"
for item in SWEEP.split(","):
    ch, ns = item.split(":")
    variants.append(dict(BSCT_CG_CHUNK=int(ch), BSCT_CHUNK_STREAMS=int(ns)))
for v in variants:
    try:
        ms, xv = run(v)
    except Exception as e:  # noqa: BLE001
        print(v, "FAILED", e, flush=True)
        continue
    same = bool(torch.equal(xv, x0))
    print(f"{v}: {ms:8.2f} ms  {ms / K * 1e3 / B:6.3f} us/slice-iter  x0 {ms0 / ms:5.3f}x  bitwise={same}  host_enqueue_ms={run.host_ms:.1f}",
          flush=True)
