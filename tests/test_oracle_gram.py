"""Pins for oracle/gram.py.

* brute force: dense continuous-y H^T H from geometric chord footprints (no box
  splines, no Toeplitz assumption) equals the Toeplitz expansion of the taps,
  column by column (north_star's check; also pins lambda_x^4 and the blur reading R1)
* closed forms: angle set {0, pi/2} (P:140 axis-aligned case) and the 45 deg case
* symmetry G[k] = G[-k] (G = H^T H symmetric), D4 symmetry for theta_i = i pi/n
* far field: R*R has the 1/|x| kernel, so the annulus mean of G pi r / n_theta -> 1
"""
import json
import os

import numpy as np
import pytest

from oracle.gram import footprint_gram_dense, gram_taps, toeplitz_matrix

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def geom(N, angles, zeta, lam=1.0):
    return dict(N=N, lambda_x=lam, angles=np.asarray(angles, float), lambda_y=1.0, n_det=3, zeta=zeta)


@pytest.mark.parametrize("zeta,lam", [(0.0, 1.0), (1.0, 1.0), (0.3, 0.5)])
def test_dense_footprint_gram(zeta, lam):
    g = geom(4, np.arange(12) * np.pi / 12, zeta, lam)
    dense = footprint_gram_dense(g)
    T = toeplitz_matrix(gram_taps(g))
    for j in range(dense.shape[1]):              # column by column
        assert np.abs(dense[:, j] - T[:, j]).max() <= 1e-12 * np.abs(T).max()


def test_irregular_angles_dense():
    rng = np.random.default_rng(3)
    g = geom(3, np.sort(rng.uniform(0, np.pi, 5)), 0.8)
    assert np.abs(footprint_gram_dense(g) - toeplitz_matrix(gram_taps(g))).max() < 1e-12


def test_axis_angles_closed_form():
    beta3 = GOLD["cubic_bspline"]["values"]
    b3 = lambda k: beta3.get(str(abs(int(k))), 0.0)
    N = 5
    d = np.arange(-(N - 1), N)
    G = gram_taps(geom(N, [0.0, np.pi / 2], 1.0))
    ref = np.array([[b3(a) + b3(b) for b in d] for a in d])
    assert np.abs(G - ref).max() < 1e-14
    G0 = gram_taps(geom(N, [0.0, np.pi / 2], 0.0))   # no blur: M_[1,1] at integers = delta
    ref0 = (d[:, None] == 0).astype(float) + (d[None, :] == 0).astype(float)
    assert np.abs(G0 - ref0).max() < 1e-14


def test_45_degrees():
    N = 4
    G = gram_taps(geom(N, [np.pi / 4], 0.0))
    assert G[N - 1, N - 1] == pytest.approx(GOLD["gram_45deg_centre"]["value"], abs=1e-14)
    beta3 = GOLD["cubic_bspline"]["values"]
    d = np.arange(-(N - 1), N)
    ref = np.array([[np.sqrt(2) * beta3.get(str(abs(b - a)), 0.0) for b in d] for a in d])
    assert np.abs(G - ref).max() < 1e-13


def test_single_axis_angle_spec():
    G = gram_taps(geom(3, [0.0], 0.0))
    assert G[2 + 1, 2] == pytest.approx(1.0, abs=1e-15)     # dk = (1, 0)
    assert G[2, 2 + 1] == pytest.approx(0.0, abs=1e-15)     # dk = (0, 1)


def test_symmetries():
    n = 24
    G = gram_taps(geom(16, np.arange(n) * np.pi / n, 1.0))
    assert np.array_equal(G, G[::-1, ::-1]) or np.abs(G - G[::-1, ::-1]).max() < 1e-15
    sc = np.abs(G).max()
    assert np.abs(G - G[::-1, :]).max() < 1e-11 * sc     # G[a,b] = G[-a,b]
    assert np.abs(G - G.T).max() < 1e-11 * sc            # G[a,b] = G[b,a]


def test_angle_shards_sum():
    g = geom(10, np.arange(30) * np.pi / 30, 0.5)
    full = gram_taps(g)
    parts = gram_taps(g, 0, 11) + gram_taps(g, 11, 17) + gram_taps(g, 17, 30)
    assert np.abs(full - parts).max() < 1e-13


def test_far_field_law():
    N, n = 128, 180
    G = gram_taps(geom(N, np.arange(n) * np.pi / n, 1.0))
    d = np.arange(-(N - 1), N)
    R = np.hypot(d[:, None], d[None, :])
    for r in (10, 20, 40, 80):
        m = (R >= r - 0.5) & (R < r + 0.5)
        assert (G[m] * np.pi * R[m] / n).mean() == pytest.approx(1.0, abs=5e-3)


@pytest.mark.parametrize("zeta,lam,n", [(0.0, 1.0, 12), (1.0, 1.0, 30), (0.5, 0.7, 17)])
def test_gram_taps_at_equals_full_filter(zeta, lam, n):
    """gram_taps_at (the sampled checker of full-size GPU filters) against the pinned full
    filter gram_taps at every offset of an N = 16 filter (irregular angles included)."""
    rng = np.random.default_rng(11)
    ang = np.concatenate([np.arange(n) * np.pi / n, rng.uniform(-1.0, 4.0, 3)])
    g = geom(16, ang, zeta, lam)
    full = gram_taps(g)
    d1, d2 = np.meshgrid(np.arange(-15, 16), np.arange(-15, 16), indexing="ij")
    from oracle.gram import gram_taps_at
    at = gram_taps_at(g, d1.ravel(), d2.ravel()).reshape(full.shape)
    assert np.abs(at - full).max() <= 1e-14 * np.abs(full).max()
