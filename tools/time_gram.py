"""Gram-filter build timings (K0 tables + K1 taps) per BASELINE config, windowed and dense.

    python tools/time_gram.py [--out profiles/r02/time_gram.json]

CUDA events around bsct_gram_build (median of 20 after 5 warm-ups), enqueued behind a ~1 ms
device sleep so that the events time the device work and not the host-side call overhead;
plan_set_filter (K0 back-projection tables + K2 spectrum) beside it."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def med_ms(fn, reps=20, warm=5):
    import numpy as np
    import torch
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)  # ~1 ms of device work: the host enqueues fn() while it runs,
        a.record()                    # so the events see device time, not Python/ctypes overhead
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    import torch

    import paper_2005_13471_b200 as bsct
    from synth import CONFIGS
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warm", type=int, default=5)
    ap.add_argument("--configs", default="1,2,3,4,5")
    a = ap.parse_args()
    bsct.load()
    rows = []
    for ci in [int(c) for c in a.configs.split(",")]:
        cfg = CONFIGS[ci]
        g = cfg.geometry()
        N = cfg.N
        dt = torch.float64 if cfg.dtype == "f64" else torch.float32
        taps = torch.empty((2 * N - 1, 2 * N - 1), dtype=dt, device="cuda")
        win = med_ms(lambda: bsct.gram_build(g, taps), a.reps, a.warm)
        os.environ["BSCT_GRAM_DENSE"] = "1"
        dense = med_ms(lambda: bsct.gram_build(g, taps), a.reps, a.warm)
        del os.environ["BSCT_GRAM_DENSE"]
        bsct.gram_build(g, taps)
        plan = bsct.plan_create(g, taps, max_batch=1)
        sf = med_ms(lambda: bsct.plan_set_filter(plan, taps), a.reps, a.warm)
        r = dict(config=ci, N=N, n_angles=cfg.n_angles, dtype=cfg.dtype, gram_build_ms=win,
                 gram_build_dense_ms=dense, set_filter_ms=sf)
        rows.append(r)
        print(json.dumps(r), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(json.dumps(r) for r in rows) + "\n")


if __name__ == "__main__":
    main()
