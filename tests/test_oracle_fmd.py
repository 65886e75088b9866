"""Pins of the FMD oracle (NEXT-2: the semi-supervised back half of Algorithm 2,
PAPER.md:268-373): transformation matrix (Eq. 7), material estimation by NNLS (Eq. 8),
mu-spectra (Eq. 9) and the Appendix-B identity."""
import itertools

import numpy as np
import pytest
from scipy.optimize import nnls as scipy_nnls


def brute_nnls(A, y):
    """Independent check: the KKT point among all passive sets (least squares on each)."""
    m = A.shape[1]
    best, bx = np.inf, None
    for r in range(m + 1):
        for P in itertools.combinations(range(m), r):
            x = np.zeros(m)
            if P:
                sol, *_ = np.linalg.lstsq(A[:, P], y, rcond=None)
                if np.any(sol < 0):
                    continue
                x[list(P)] = sol
            f = np.sum((A @ x - y) ** 2)
            if f < best - 1e-15:
                best, bx = f, x
    return bx


@pytest.mark.parametrize("rows,m,seed", [(6, 3, 0), (8, 5, 1), (5, 5, 2), (12, 8, 3), (3, 1, 4)])
def test_nnls_matches_scipy_and_brute_force(orc, rows, m, seed):
    g = np.random.default_rng(seed)
    for trial in range(20):
        A = g.normal(size=(rows, m)) + 0.3
        y = g.normal(size=rows)
        x = orc.nnls(A, y)
        xs, _ = scipy_nnls(A, y)
        np.testing.assert_allclose(x, xs, atol=1e-10)
        np.testing.assert_allclose(x, brute_nnls(A, y), atol=1e-10)


def test_nnls_kkt(orc):
    g = np.random.default_rng(7)
    for _ in range(50):
        A = g.random(size=(6, 4))
        y = g.normal(size=6)
        x = orc.nnls(A, y)
        grad = A.T @ (A @ x - y)
        assert np.all(x >= 0)
        assert np.all(grad >= -1e-10)
        assert np.allclose(x * grad, 0, atol=1e-10)


def test_nnls_interior_equals_least_squares(orc):
    g = np.random.default_rng(8)
    A = g.random(size=(7, 3)) + 0.5
    xt = np.array([0.7, 1.3, 0.2])
    x = orc.nnls(A, A @ xt)
    np.testing.assert_allclose(x, xt, atol=1e-12)


def test_transform_is_region_mean(orc):
    g = np.random.default_rng(9)
    K, Nx, Nm = 5, 400, 3
    X = g.random((K, Nx))
    lab = g.integers(-1, Nm, Nx).astype(np.int32)
    T, cnt = orc.fmd_transform(X, lab, Nm)
    for i in range(Nm):
        sel = lab == i
        assert cnt[i] == sel.sum()
        np.testing.assert_allclose(T[i], X[:, sel].mean(axis=1), rtol=1e-13)


def test_transform_errors(orc):
    X = np.ones((2, 10))
    with pytest.raises(ValueError):
        orc.fmd_transform(X, np.full(10, 0, np.int32), 2)  # region 1 empty
    with pytest.raises(ValueError):
        orc.fmd_transform(X, np.full(10, 3, np.int32), 2)  # label out of range


def mixture_problem(g, K=6, Nm=3, Nx=500):
    """x^s = x^m T exactly with x^m >= 0: pure regions (one material, fraction 1) plus
    mixed and empty voxels."""
    T = g.random((Nm, K)) + 0.2
    xm = np.zeros((Nm, Nx))
    lab = np.full(Nx, -1, np.int32)
    for n in range(Nx):
        kind = n % 5
        if kind < Nm:                        # pure voxel of material `kind`
            xm[kind, n] = 1.0
            lab[n] = kind
        elif kind == Nm:                     # mixture
            xm[:, n] = g.random(Nm) * (g.random(Nm) > 0.3)
    X = T.T @ xm                             # [K, Nx]
    return T, xm, lab, X


def test_materials_recover_exact_mixtures(orc):
    g = np.random.default_rng(10)
    T, xm, lab, X = mixture_problem(g)
    T2, _ = orc.fmd_transform(X, lab, T.shape[0])
    np.testing.assert_allclose(T2, T, rtol=1e-13)          # pure regions -> exact T (Eq. 7)
    Xm = orc.fmd_materials(X, T2)
    np.testing.assert_allclose(Xm, xm, atol=1e-11)


def test_materials_match_scipy_per_voxel(orc):
    g = np.random.default_rng(11)
    K, Nm, Nx = 5, 3, 200
    T = g.random((Nm, K)) + 0.1
    X = g.normal(size=(K, Nx))
    Xm = orc.fmd_materials(X, T)
    for n in range(Nx):
        np.testing.assert_allclose(Xm[:, n], scipy_nnls(T.T, X[:, n])[0], atol=1e-10)


def test_spectra_and_appendix_b_identity(orc):
    """D^m = D^s T^T (Eq. 9); with x^s = x^m T: x^s (D^s)^T = x^m (D^m)^T (Appendix B)."""
    g = np.random.default_rng(12)
    T, xm, lab, X = mixture_problem(g, K=4, Nm=2, Nx=100)
    D = g.random((4, 37))
    Dm = orc.fmd_spectra(D, T)
    np.testing.assert_allclose(Dm, T @ D, rtol=1e-13)
    Xm = orc.fmd_materials(X, orc.fmd_transform(X, lab, 2)[0])
    Xh_sub = orc.synthesize(X.reshape(4, 1, 10, 10), D)
    Xh_mat = orc.synthesize(Xm.reshape(2, 1, 10, 10), Dm)
    np.testing.assert_allclose(Xh_mat, Xh_sub, rtol=1e-10, atol=1e-12)
