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


def _dense_G(taps, N):
    from oracle.normal import apply_direct
    cols = []
    for k in range(N * N):
        e = np.zeros((N, N))
        e.flat[k] = 1.0
        cols.append(apply_direct(taps, e).ravel())
    return np.stack(cols, axis=1)


def test_chebyshev_residual_polynomial():
    """r_k = T_k((theta - G)/delta) b / T_k(theta/delta) (Chebyshev polynomial identity, checked
    through the eigendecomposition of the dense Toeplitz operator), and the minimax bound
    ||r_k|| <= ||b|| / T_k(theta/delta) when the spectrum lies in [lmin, lmax]."""
    from numpy.polynomial import chebyshev as C
    from oracle.gram import gram_taps
    from oracle.solvers import chebyshev
    g = dict(N=6, lambda_x=1.0, angles=np.arange(12) * np.pi / 12, lambda_y=1.0, n_det=13, zeta=1.0)
    T = gram_taps(g)
    G = _dense_G(T, 6)
    lam, V = np.linalg.eigh(G)
    b = np.random.default_rng(4).standard_normal((6, 6))
    for lmin, lmax in ((lam[0], lam[-1]), (0.5 * lam[0], 1.2 * lam[-1])):
        theta, delta = 0.5 * (lmax + lmin), 0.5 * (lmax - lmin)
        for k in (1, 3, 7):
            x, hist = chebyshev(T, b, k, lmin, lmax, direct=True)
            ck = np.zeros(k + 1)
            ck[k] = 1.0
            pk = C.chebval((theta - lam) / delta, ck) / C.chebval(theta / delta, ck)
            r_pred = V @ (pk * (V.T @ b.ravel()))
            r = b.ravel() - G @ x.ravel()
            assert np.abs(r - r_pred).max() < 1e-10 * np.abs(b).max()
            assert hist[-1] <= np.linalg.norm(b) / C.chebval(theta / delta, ck) * (1 + 1e-10)


def test_chebyshev_exact_interval_one_point():
    """lmin = lmax = G00 on N = 1: d0 = b / G00 and x_1 = b / G00 exactly."""
    from oracle.gram import gram_taps
    from oracle.solvers import chebyshev
    g = dict(N=1, lambda_x=1.0, angles=np.arange(4) * np.pi / 4, lambda_y=1.0, n_det=5, zeta=0.0)
    T = gram_taps(g)
    lam = float(T[0, 0])
    x, _ = chebyshev(T, np.array([[3.0]]), 1, lam * (1 - 1e-9), lam * (1 + 1e-9), direct=True)
    assert x[0, 0] == pytest.approx(3.0 / lam, rel=1e-8)
