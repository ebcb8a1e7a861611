"""Pins for oracle/backproject.py (Eq.(5))."""
import json
import os

import numpy as np
import pytest

from oracle.backproject import (H_CORR, backproject, backproject_quadrature, correction_filter,
                                corrected_row, interpolant, interpolation_degree)
from oracle.boxspline import box_spline
from oracle.forward import forward
from oracle.gram import gram_taps
from oracle.normal import apply_direct

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_q40_paper_value():
    q = correction_filter(2, h=45)
    assert q[45 + 40] == pytest.approx(GOLD["q40"]["value"], rel=GOLD["q40"]["rel_tol"])
    assert q[45 - 40] == q[45 + 40]


def test_q_inverts_b():
    """Eq.(5): Q(z) = 1/B(z), b[m] = <delta(y - m), B(y)> = B_2(m) = M_[1,1,1](m)."""
    b = box_spline([1.0, 1.0, 1.0], np.array([-1.0, 0.0, 1.0]))
    assert np.allclose(b, [1 / 8, 6 / 8, 1 / 8], atol=1e-15)
    q = correction_filter(2)
    qb = np.convolve(q, b)[1:-1]
    delta = (np.arange(2 * H_CORR + 1) == H_CORR).astype(float)
    assert np.abs(qb - delta)[5:-5].max() < 1e-15
    assert np.abs(qb - delta).max() < 1e-12             # truncation at h = 25: |q[26]| ~ 1e-20
    assert np.array_equal(correction_filter(1), delta)  # q = delta for degree 0/1
    assert np.array_equal(correction_filter(0), delta)


def test_degree_rule():
    g = dict(N=4, lambda_x=1.0, angles=[0.0], lambda_y=1.0, n_det=5, zeta=0.0)
    assert interpolation_degree(g, np.pi / 6) == 1           # C^0
    assert interpolation_degree(g, np.pi / 2) == 0           # axis aligned C^-1
    assert interpolation_degree(g, 0.0) == 0
    g["zeta"] = 1.0
    assert interpolation_degree(g, np.pi / 6) == 2           # blur C^1
    assert interpolation_degree(g, np.pi / 2) == 1           # blur, axis C^0


@pytest.mark.parametrize("zeta,t", [(0.0, 0.3), (0.0, 0.0), (1.0, 0.3), (1.0, np.pi / 2)])
def test_interpolant_reproduces_samples(zeta, t):
    """Oblique projection with the correction filter interpolates: g^(y_m) = g_s[m]
    (P:141-143), away from the zero-extension edges."""
    M = 40
    g = dict(N=4, lambda_x=1.0, angles=[t], lambda_y=1.0, n_det=M, zeta=zeta)
    row = np.random.default_rng(5).standard_normal(M)
    y = 1.0 * (np.arange(M) - M // 2)
    gh = interpolant(g, t, row, y)
    assert np.abs(gh - row)[3:-3].max() < 1e-12


def test_closed_form_equals_quadrature():
    g = dict(N=5, lambda_x=1.0, angles=np.arange(7) * np.pi / 7, lambda_y=1.0, n_det=11, zeta=0.7)
    sino = np.random.default_rng(6).standard_normal((7, 11))
    b = backproject(g, sino)
    for (k1, k2) in [(1, 3), (2, 2), (4, 0)]:
        q = backproject_quadrature(g, sino, k1, k2)
        assert abs(q - b[k1, k2]) < 1e-6 * np.abs(b).max()


def test_closed_form_quadrature_lambda_y():
    g = dict(N=4, lambda_x=1.0, angles=np.array([0.2, 1.1, np.pi / 2]), lambda_y=0.5, n_det=21, zeta=0.5)
    sino = np.random.default_rng(7).standard_normal((3, 21))
    b = backproject(g, sino)
    q = backproject_quadrature(g, sino, 1, 2)
    assert abs(q - b[1, 2]) < 1e-6 * np.abs(b).max()


@pytest.mark.parametrize("zeta", [0.0, 1.0])
def test_exact_recovery_axis_angles(zeta):
    """the signal is recovered exactly when all k_theta are sampling points, so
    H^T g^ of a forward projection equals G c at angles {0, pi/2}, lambda_y = lambda_x."""
    N = 6
    g = dict(N=N, lambda_x=1.0, angles=np.array([0.0, np.pi / 2]), lambda_y=1.0, n_det=15, zeta=zeta)
    c = np.random.default_rng(8).standard_normal((N, N))
    b = backproject(g, forward(g, c))
    y = apply_direct(gram_taps(g), c)
    assert np.abs(b - y).max() < 1e-13 * np.abs(y).max()


def test_spec_single_bin():
    """single angle 0, one nonzero centre bin -> column k_theta = 0 gets 1."""
    N = 5
    g = dict(N=N, lambda_x=1.0, angles=np.array([0.0]), lambda_y=1.0, n_det=9, zeta=0.0)
    s = np.zeros((1, 9))
    s[0, 4] = 1.0
    b = backproject(g, s)
    ref = np.zeros((N, N))
    ref[:, N // 2] = 1.0
    assert np.abs(b - ref).max() < 1e-15


def test_corrected_row_layout():
    row = np.arange(1.0, 6.0)
    assert np.array_equal(corrected_row(row, 1)[H_CORR:H_CORR + 5], row)
    full = corrected_row(row, 2)
    assert full.shape == (5 + 2 * H_CORR,)
    assert full[H_CORR + 2] == pytest.approx(np.dot(row, correction_filter(2)[H_CORR + 2 - np.arange(5)]))


@pytest.mark.parametrize("zeta,ly,n_det", [(1.0, 1.0, 25), (0.0, 0.5, 47), (1.5, 1.0, 20), (0.5, 0.75, 31)])
def test_backproject_pixels_equals_full(zeta, ly, n_det):
    """backproject(pixels=...) (the sampled checker of full-size GPU back projections) against
    the full-grid backproject at every pixel of an N = 16 image, in a shuffled pixel order."""
    rng = np.random.default_rng(5)
    ang = np.concatenate([np.arange(24) * np.pi / 24, rng.uniform(0, np.pi, 3)])
    g = dict(N=16, lambda_x=1.0, angles=ang, lambda_y=ly, n_det=n_det, zeta=zeta)
    sino = rng.uniform(-1, 1, (len(ang), n_det))
    full = backproject(g, sino)
    k1, k2 = np.meshgrid(np.arange(16), np.arange(16), indexing="ij")
    perm = rng.permutation(256)
    k1, k2 = k1.ravel()[perm], k2.ravel()[perm]
    at = backproject(g, sino, pixels=(k1, k2))
    assert np.abs(at - full[k1, k2]).max() <= 1e-14 * np.abs(full).max()
