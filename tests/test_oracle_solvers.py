"""Pins for oracle/solvers.py: textbook CG / SD / Landweber properties
and convergence to the dense direct solve (numpy.linalg on the expanded Toeplitz G)."""
import numpy as np
import pytest

from oracle import solvers
from oracle.gram import gram_taps, toeplitz_matrix
from oracle.normal import apply_direct


def problem(N=8, n=16, zeta=1.0, seed=0):
    T = gram_taps(dict(N=N, lambda_x=1.0, angles=np.arange(n) * np.pi / n, lambda_y=1.0, n_det=3, zeta=zeta))
    b = np.random.default_rng(seed).standard_normal((N, N))
    return T, b


def test_single_pixel_one_step():
    T, b = problem(N=1)
    x, h = solvers.cg(T, b, 1)
    assert x[0, 0] == pytest.approx(b[0, 0] / T[0, 0], rel=1e-15)
    x, h = solvers.sd(T, b, 1)
    assert x[0, 0] == pytest.approx(b[0, 0] / T[0, 0], rel=1e-15)


def test_cg_converges_to_dense_solve():
    T, b = problem()
    ref = np.linalg.solve(toeplitz_matrix(T), b.ravel()).reshape(b.shape)
    x, h = solvers.cg(T, b, 200, direct=True)
    assert np.linalg.norm(x - ref) < 1e-6 * np.linalg.norm(ref)


def test_cg_orthogonality_and_monotone():
    T, b = problem(seed=1)
    rec = []
    x, h = solvers.cg(T, b, 6, record=rec)   # before rounding erodes orthogonality
    rs = [b - apply_direct(T, r["x"]) for r in rec]
    for i in range(len(rs)):
        for j in range(i):
            assert abs(np.vdot(rs[i], rs[j])) < 1e-10 * np.linalg.norm(rs[i]) * np.linalg.norm(rs[j]) + 1e-12
    f = [solvers.objective(T, b, r["x"]) for r in rec]
    assert all(f[i + 1] <= f[i] + 1e-12 * abs(f[i]) for i in range(len(f) - 1))


def test_sd_orthogonality_monotone_convergence():
    T, b = problem(seed=2)
    r_prev = b
    x = np.zeros_like(b)
    f_prev = 0.0
    for k in range(1, 15):
        xk, _ = solvers.sd(T, b, k, direct=True)
        rk = b - apply_direct(T, xk)
        if k > 1:
            assert abs(np.vdot(rk, r_prev)) < 1e-8 * np.linalg.norm(rk) * np.linalg.norm(r_prev)
        f = solvers.objective(T, b, xk)
        assert f < f_prev
        r_prev, f_prev = rk, f
    ref = np.linalg.solve(toeplitz_matrix(T), b.ravel()).reshape(b.shape)
    xs, _ = solvers.sd(T, b, 3000)
    assert np.linalg.norm(xs - ref) < 1e-4 * np.linalg.norm(ref)


def test_landweber():
    T, b = problem(seed=3)
    tau = solvers.landweber_tau(T)
    lam_max = np.linalg.eigvalsh(toeplitz_matrix(T)).max()
    assert tau * lam_max <= 1.0 + 1e-12         # interlacing: Toeplitz <= circulant embedding
    x, h = solvers.landweber(T, b, 50)
    assert np.all(np.diff(h) <= 1e-12)          # residual non-increasing for tau <= 1/lambda_max
    xd, _ = solvers.landweber(T, b, 5, direct=True)
    xf, _ = solvers.landweber(T, b, 5)
    assert np.abs(xd - xf).max() < 1e-12


def test_zero_rhs():
    T, b = problem()
    x, h = solvers.cg(T, np.zeros_like(b), 5)
    assert not x.any() and not h.any()
