"""NEXT-3 harness (tools/experiments.py) runs end to end through the library on a tiny case."""
import math
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def test_quality_sweep_tiny(cuda_lib):
    import experiments
    rows = experiments.run(N=32, n_views=30, ratios=(0.5, 1.0), noise=(0.0, 0.01), iters=10)
    assert len(rows) == 2 * 2 * 2 * 2
    for r in rows:
        assert math.isfinite(r["snr_db"]) and r["snr_db"] > 3.0, r
    md = experiments.to_markdown(rows, 32, 10)
    assert md.count("\n| ") == 1 + 2 * 2 * 2  # header + one row per (ratio, noise, solver)


@pytest.mark.parametrize("ratio,zeta", [(1.0, 1.0), (0.5, 0.0)])
def test_metrics_match_oracle_reconstruction(cuda_lib, ratio, zeta):
    """SNR and SSIM of one GPU reconstruction (steepest descent) against the same metrics
    of the FP64 oracle's reconstruction from the same sinogram (oracle Gram filter, back
    projection and SD; SD keeps FP32/FP64 parity)."""
    import experiments
    from oracle import solvers
    from oracle.backproject import backproject
    from oracle.gram import gram_taps
    ref, sino, g0 = experiments.problem(48, 60, ratio, 0.01, 2000)
    g = dict(g0, zeta=zeta * ratio)
    x = experiments.reconstruct_gpu(g, sino, ("sd",), 20)["sd"]
    xo, _ = solvers.sd(gram_taps(g), backproject(g, sino), 20)
    assert experiments.snr_db(ref, x) == pytest.approx(experiments.snr_db(ref, xo), abs=1e-3)
    assert experiments.ssim(ref, x) == pytest.approx(experiments.ssim(ref, xo), abs=1e-4)
