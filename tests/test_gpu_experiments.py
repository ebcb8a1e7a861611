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
