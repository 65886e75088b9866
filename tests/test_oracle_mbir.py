"""Pins of the MBIR oracle (NEXT-3: Eq. 5, with the QGGMRF prior and the SQS
iteration of DESIGN.md R24-R26), CPU only.

* QGGMRF: rho'(d) = w(d) d agrees with a central difference of rho; rho is even, rho(0) = 0;
  w(0) has the closed form q / (p sx^p (T sx)^(q-p)); for |d| >> T sx, rho -> |d|^p / (p sx^p).
* The projector is the matrix A re-derived here independently (numpy: weights
  max(0, 1 - |u - c|)), and the backprojector is exactly A^T.
* SQS is a majorize-minimize iteration: the Eq. 5 objective never increases.
* With the prior switched off (sx huge), the iterates converge to the non-negative least-squares
  solution (scipy.optimize.nnls on the explicit A); with y = A x*, x* > 0, to x* itself.
* A constant image with y = A x0 is a fixed point (zero data gradient, zero prior gradient).
"""
import math

import numpy as np
import pytest
from scipy.optimize import nnls

import oracle


def explicit_A(nc, nv):
    """A[(v, c), (i, j)] = max(0, 1 - |u_ij(v) - c|), u = x_j cos + y_i sin + (nc-1)/2,
    x_j = j - (nc-1)/2, y_i = i - (nc-1)/2, theta_v = v pi / nv."""
    half = 0.5 * (nc - 1)
    A = np.zeros((nv * nc, nc * nc))
    for v in range(nv):
        th = v * math.pi / nv
        for i in range(nc):
            for j in range(nc):
                u = (j - half) * math.cos(th) + (i - half) * math.sin(th) + half
                for c in range(nc):
                    A[v * nc + c, i * nc + j] = max(0.0, 1.0 - abs(u - c))
    return A


def test_qggmrf_potential():
    prm = oracle.mbir_params(1.0, 0.7, p=1.2, q=2.0, T=1.3)
    for d in (-3.0, -0.4, -1e-3, 2e-3, 0.05, 0.9, 5.0):
        h = 1e-6 * max(1.0, abs(d))
        fd = (oracle.qggmrf_rho(d + h, prm) - oracle.qggmrf_rho(d - h, prm)) / (2 * h)
        assert abs(fd - oracle.qggmrf_omega(d, prm) * d) <= 1e-6 * max(1.0, abs(fd))
        assert oracle.qggmrf_rho(d, prm) == pytest.approx(oracle.qggmrf_rho(-d, prm), rel=1e-15)
        assert oracle.qggmrf_rho(d, prm) >= 0.0
    assert oracle.qggmrf_rho(0.0, prm) == 0.0
    sx, p, q, T = 0.7, 1.2, 2.0, 1.3
    assert oracle.qggmrf_omega(0.0, prm) == pytest.approx(q / (p * sx ** p * (T * sx) ** (q - p)), rel=1e-14)
    d = 1e4
    assert oracle.qggmrf_rho(d, prm) == pytest.approx(d ** p / (p * sx ** p), rel=1e-3)
    # w non-increasing in |d| (what the half-quadratic surrogate needs)
    ws = [oracle.qggmrf_omega(x, prm) for x in np.linspace(0, 10, 200)]
    assert all(a >= b for a, b in zip(ws, ws[1:]))


def test_projector_is_the_explicit_matrix_and_backprojector_its_transpose():
    nc, nv = 9, 7
    A = explicit_A(nc, nv)
    rng = np.random.default_rng(1)
    x = rng.random((nc, nc))
    r = rng.standard_normal((nv, nc))
    assert np.allclose(oracle.mbir_project_slice(x, nv), (A @ x.reshape(-1)).reshape(nv, nc), rtol=0, atol=1e-12)
    assert np.allclose(oracle.mbir_backproject_slice(r), (A.T @ r.reshape(-1)).reshape(nc, nc), rtol=0, atol=1e-12)


@pytest.mark.parametrize("sv,sx,p", [(1.0, 0.5, 1.2), (0.3, 2.0, 1.0), (2.0, 0.1, 2.0)])
def test_sqs_objective_never_increases(sv, sx, p):
    nc, nv = 16, 12
    rng = np.random.default_rng(int(100 * sv + 10 * sx))
    xt = rng.random((nc, nc))
    y = oracle.mbir_project_slice(xt, nv) + 0.3 * rng.standard_normal((nv, nc))
    x, obj = oracle.mbir_slice(y, rng.random((nc, nc)), oracle.mbir_params(sv, sx, p=p), 40, objective=True)
    assert np.all(np.diff(obj) <= 1e-12 * np.abs(obj[:-1]))
    assert obj[-1] < obj[0] and np.all(x >= 0)


def test_prior_off_converges_to_nnls():
    # a small, moderately conditioned system (cond(A) ~ 1e2) so that 4000 SQS iterations
    # reach the NNLS minimiser to ~1e-10 (larger images converge too, but slowly)
    nc, nv = 4, 8
    A = explicit_A(nc, nv)
    rng = np.random.default_rng(3)
    y = A @ rng.random(nc * nc) + 0.2 * rng.standard_normal(nv * nc)
    x_ref, _ = nnls(A, y)
    prm = oracle.mbir_params(1.0, 1e6)   # prior weight ~ 1e-12: the data term alone
    x = oracle.mbir_slice(y.reshape(nv, nc), np.full((nc, nc), 0.5), prm, 4000)
    assert np.linalg.norm(x.reshape(-1) - x_ref) <= 1e-6 * np.linalg.norm(x_ref)
    assert (x_ref == 0).any()   # the non-negativity constraint is active at the solution


def test_prior_off_recovers_exact_solution():
    # 3x3 image, 8 views: A has full column rank and SQS contracts fast enough to reach x*
    nc, nv = 3, 8
    A = explicit_A(nc, nv)
    xs = np.random.default_rng(4).random(nc * nc) + 0.5
    y = (A @ xs).reshape(nv, nc)
    x = oracle.mbir_slice(y, np.ones((nc, nc)), oracle.mbir_params(1.0, 1e6), 4000)
    assert np.linalg.norm(x.reshape(-1) - xs) <= 1e-6 * np.linalg.norm(xs)


def test_constant_image_is_a_fixed_point():
    nc, nv = 12, 10
    x0 = np.full((nc, nc), 0.37)
    y = oracle.mbir_project_slice(x0, nv)
    x = oracle.mbir_slice(y, x0, oracle.mbir_params(0.5, 0.2), 5)
    assert np.allclose(x, x0, rtol=0, atol=1e-13)


def test_multi_channel_driver_matches_per_slice():
    Nv, Nr, Nc, K = 8, 2, 10, 2
    rng = np.random.default_rng(5)
    V = rng.random((Nv * Nr * Nc, K))
    X0 = rng.random((K, Nr, Nc, Nc))
    prm = oracle.mbir_params(1.0, 0.3)
    X = oracle.mbir(V, Nv, Nr, Nc, X0, prm, 6)
    Vr = V.reshape(Nv, Nr, Nc, K)
    for k in range(K):
        for r in range(Nr):
            assert np.array_equal(X[k, r], oracle.mbir_slice(Vr[:, r, :, k], X0[k, r], prm, 6))
