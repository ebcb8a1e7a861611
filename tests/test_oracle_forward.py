"""Pins for oracle/forward.py (Eq.(3), Eq.(4)): geometric footprints,
mass conservation and SPEC's single-pixel examples."""
import numpy as np
import pytest

from oracle.forward import forward, forward_geometric


@pytest.mark.parametrize("zeta,lam", [(0.0, 1.0), (0.7, 1.0), (0.4, 0.5)])
def test_forward_equals_geometric(zeta, lam):
    g = dict(N=5, lambda_x=lam, angles=np.arange(7) * np.pi / 7 + 0.05, lambda_y=0.8, n_det=13, zeta=zeta)
    c = np.random.default_rng(9).standard_normal((5, 5))
    a, b = forward(g, c), forward_geometric(g, c)
    assert np.abs(a - b).max() < 1e-12 * np.abs(a).max()


def test_mass_conservation():
    """lambda_y sum_m g[theta, m] = lambda_x^2 sum c, exact when the detector
    width is 1 = lambda_y (the blur box is a partition of unity on the integer grid)."""
    N = 6
    g = dict(N=N, lambda_x=1.0, angles=np.arange(9) * np.pi / 9, lambda_y=1.0, n_det=21, zeta=1.0)
    c = np.random.default_rng(10).uniform(0, 1, (N, N))
    s = forward(g, c)
    assert np.abs(s.sum(axis=1) - c.sum()).max() < 1e-12


def test_single_pixel_spec():
    one = np.ones((1, 1))
    g = dict(N=1, lambda_x=1.0, angles=np.array([0.0, np.pi / 4]), lambda_y=0.75, n_det=3, zeta=0.0)
    s = forward(g, one)   # detector y = -0.75, 0, 0.75
    assert s[0, 1] == pytest.approx(1.0) and s[0, 2] == 0.0
    assert s[1, 1] == pytest.approx(np.sqrt(2.0), abs=1e-14)
    g = dict(N=1, lambda_x=1.0, angles=np.array([0.0]), lambda_y=1.0, n_det=3, zeta=1.0)
    s = forward(g, one)
    assert s[0, 1] == pytest.approx(1.0) and s[0, 0] == 0.0 and s[0, 2] == 0.0
