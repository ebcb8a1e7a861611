"""K4 v4 (tensor cores) against K4 v3 (CUDA cores) on the same inputs: relative L2 difference and
device time per launch.  BSCT_BP_V3=1 selects v3 at plan creation."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2005_13471_b200 as bsct
    bsct.load()
    cases = [(100, 60, 151, 1.0, 3), (512, 360, 725, 1.0, 130), (256, 180, 363, 1.0, 16), (512, 360, 725, 1.5, 8)]
    if len(sys.argv) > 1:
        cases = [(512, 360, 725, 1.0, int(sys.argv[1]))]
    for N, n, M, zeta, B in cases:
        g = dict(N=N, lambda_x=1.0, angles=np.arange(n) * np.pi / n, lambda_y=1.0, n_det=M, zeta=zeta)
        taps = torch.empty((2 * N - 1, 2 * N - 1), device="cuda")
        bsct.gram_build(g, taps)
        gen = torch.Generator(device="cuda").manual_seed(N + B)
        sino = torch.rand((B, n, M), device="cuda", generator=gen)
        res, ts = {}, {}
        for v3 in ("1", "0"):
            os.environ["BSCT_BP_V3"] = v3
            plan = bsct.plan_create(g, taps, max_batch=B)
            b = torch.empty((B, N, N), device="cuda")
            bsct.backproject(plan, sino, b)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                bsct.backproject(plan, sino, b)
            e1.record()
            torch.cuda.synchronize()
            res[v3], ts[v3] = b.clone(), e0.elapsed_time(e1) / 3
            del plan
        d = float((res["0"] - res["1"]).norm() / res["1"].norm())
        print(f"N={N} n={n} B={B} zeta={zeta}: rel_l2(v4, v3) = {d:.3e}; v3 {ts['1']:.3f} ms, v4 {ts['0']:.3f} ms "
              f"({B * N * N * n / (ts['0'] / 1e3) / 1e9:.0f} Gvox-angle/s)", flush=True)


if __name__ == "__main__":
    main()
