"""Pins for the oracle's NMF (oracle.c: oracle_nmf) against things other than itself.

Eq. 4 solved by Lee-Seung multiplicative updates (DESIGN.md
R1-R3).  Each pin is chosen so a plausible mistake (dropped term, wrong index,
transposed operand, wrong update order) fails at least one of them:

* golden worked example (hand-derived rationals, tests/golden/) -- order, indices;
* K = 1 reduces MU to the power method on Y^T Y (closed form, numpy matmul /
  LAPACK SVD as the independent route);
* rank-1 data are factorised exactly after one iteration;
* exact fixed point on integer-valued V* D*;
* scale and permutation equivariances;
* Lee & Seung's monotonicity theorem for the objective;
* exact recovery of noiseless rank-N_m data (Eq. 3 with w = 0);
* the Gram identity for the objective.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import synthdata as sd

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _frac(x):
    return float(Fraction(str(x)))


def test_worked_example_golden(orc):
    g = json.load(open(os.path.join(GOLD, "nmf_worked_example.json")))
    Y = np.array(g["Y"], dtype=np.float32)
    V0 = np.array(g["V0"], dtype=np.float64)
    D0 = np.array(g["D0"], dtype=np.float64)
    assert orc.nmf_objective(Y, V0, D0) == pytest.approx(_frac(g["objective0"]), abs=1e-15)
    V1, D1, obj = orc.nmf(Y, V0, D0, 1, objective=True)
    np.testing.assert_allclose(V1, [[_frac(v[0])] for v in g["V1"]], rtol=0, atol=1e-15)
    np.testing.assert_allclose(D1, [[_frac(d) for d in g["D1"][0]]], rtol=0, atol=1e-15)
    assert obj[0] == pytest.approx(_frac(g["objective_after_V1"]), abs=1e-14)
    assert obj[1] == pytest.approx(_frac(g["objective_after_D1"]), abs=1e-14)


def test_k1_is_power_iteration(orc):
    """K = 1: V <- Y D^T/||D||^2 and D <- V^T Y/||V||^2, so
    D_{n+1} = D_n (Y^T Y) ||D_n||^2 / ||Y D_n^T||^2 (power method on Y^T Y)."""
    rng = np.random.default_rng(7)
    Y = rng.uniform(0, 1, size=(37, 11)).astype(np.float32)
    Yd = Y.astype(np.float64)
    V0 = rng.uniform(0.5, 1.5, size=(37, 1))
    D0 = rng.uniform(0.5, 1.5, size=(1, 11))
    n = 6
    V, D = orc.nmf(Y, V0, D0, n)
    d = D0.copy()
    M = Yd.T @ Yd
    for _ in range(n):
        d = (d @ M) * (d @ d.T).item() / float(np.sum((Yd @ d.T) ** 2))
    v_last = None
    # V_n = Y D_{n-1}^T / ||D_{n-1}||^2
    dprev = D0.copy()
    for _ in range(n - 1):
        dprev = (dprev @ M) * (dprev @ dprev.T).item() / float(np.sum((Yd @ dprev.T) ** 2))
    v_last = Yd @ dprev.T / (dprev @ dprev.T).item()
    np.testing.assert_allclose(D, d, rtol=1e-12)
    np.testing.assert_allclose(V, v_last, rtol=1e-12)


def test_k1_converges_to_top_singular_pair(orc):
    rng = np.random.default_rng(3)
    Y = rng.uniform(0, 1, size=(30, 9)).astype(np.float32)
    V, D = orc.nmf(Y, np.ones((30, 1)), np.ones((1, 9)), 200)
    U, S, Wt = np.linalg.svd(Y.astype(np.float64))
    w = Wt[0] * np.sign(Wt[0].sum())
    np.testing.assert_allclose(D[0] / np.linalg.norm(D), w, atol=1e-12)
    assert np.linalg.norm(V) * np.linalg.norm(D) == pytest.approx(S[0], rel=1e-12)


def test_rank1_exact_after_one_iteration(orc):
    u = np.array([1, 2, 3, 4, 5], dtype=np.float64)
    w = np.array([2, 1, 0.5, 4], dtype=np.float64)
    Y = np.outer(u, w).astype(np.float32)  # exact in fp32
    V, D = orc.nmf(Y, np.full((5, 1), 0.3), np.full((1, 4), 1.7), 1)
    np.testing.assert_allclose(V @ D, Y, rtol=1e-14)


def test_fixed_point_integer_factorisation(orc):
    rng = np.random.default_rng(11)
    Vs = rng.integers(1, 5, size=(20, 3)).astype(np.float64)
    Ds = rng.integers(1, 5, size=(3, 13)).astype(np.float64)
    Y = (Vs @ Ds).astype(np.float32)  # small integers: exact in fp32
    V, D, obj = orc.nmf(Y, Vs, Ds, 10, objective=True)
    np.testing.assert_allclose(V, Vs, rtol=1e-14)
    np.testing.assert_allclose(D, Ds, rtol=1e-14)
    assert np.all(obj < 1e-20)


def test_scale_equivariance(orc):
    pr = sd.make_problem(sd.custom(Nc=16, Nv=12, Nk=30, K=3, M=3))
    Y, V0, D0 = pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy()
    V, D = orc.nmf(Y, V0, D0, 15)
    V2, D2 = orc.nmf(Y, 2.0 * V0.astype(np.float64), D0.astype(np.float64) / 2.0, 15)
    np.testing.assert_allclose(V2, 2.0 * V, rtol=1e-13)
    np.testing.assert_allclose(D2, D / 2.0, rtol=1e-13)


def test_permutation_equivariance(orc):
    pr = sd.make_problem(sd.custom(Nc=16, Nv=12, Nk=30, K=3, M=3))
    Y, V0, D0 = pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy()
    V, D = orc.nmf(Y, V0, D0, 12)
    rng = np.random.default_rng(5)
    pr_ = rng.permutation(Y.shape[0])
    pb = rng.permutation(Y.shape[1])
    pk = rng.permutation(3)
    Vp, Dp = orc.nmf(Y[pr_][:, pb], V0[pr_][:, pk], D0[pk][:, pb], 12)
    np.testing.assert_allclose(Vp, V[pr_][:, pk], rtol=1e-10)
    np.testing.assert_allclose(Dp, D[pk][:, pb], rtol=1e-10)


def test_monotone_objective(orc):
    pr = sd.make_problem(sd.CONFIGS[1])
    Y, V0, D0 = pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy()
    _, _, obj = orc.nmf(Y, V0, D0, 40, objective=True)
    f0 = orc.nmf_objective(Y, V0, D0)
    seq = np.concatenate([[f0], obj])
    assert np.all(np.diff(seq) <= 1e-12 * seq[:-1]), np.diff(seq).max()
    assert seq[-1] < 0.5 * seq[0]


def test_gram_identity(orc):
    pr = sd.make_problem(sd.custom(Nc=16, Nv=12, Nk=30, K=3, M=3))
    Y = pr["Y"].numpy().astype(np.float64)
    V, D = orc.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), 5)
    Yp = np.maximum(Y, 0)
    gram = (Yp * Yp).sum() - 2 * np.sum((V.T @ Yp) * D) + np.sum((V.T @ V) * (D @ D.T))
    assert orc.nmf_objective(pr["Y"].numpy(), V, D) == pytest.approx(gram, rel=1e-11)


def test_clamp_of_negative_data(orc):
    """Y enters the NMF as Y+ = max(Y, 0) (R6): negating the negative entries changes nothing."""
    rng = np.random.default_rng(2)
    Y = rng.normal(0.3, 0.5, size=(25, 8)).astype(np.float32)
    Yc = np.maximum(Y, 0)
    V0 = rng.uniform(0.5, 1, size=(25, 2))
    D0 = rng.uniform(0.5, 1, size=(2, 8))
    a = orc.nmf(Y, V0, D0, 5)
    b = orc.nmf(Yc, V0, D0, 5)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


def test_exact_recovery_noiseless_rank_m(orc):
    """Eq. 3 with w = 0 is exactly rank N_m: the residual of the product V D
    (not the factors, R8) goes to ~0."""
    cfg = sd.custom(idx=1, Nc=32, Nv=45, Nk=200, K=3, M=3)
    pr = sd.make_problem(cfg, noise=False)
    Y = pr["Y"].numpy()
    V, D = orc.nmf(Y, pr["V0"].numpy(), pr["D0"].numpy(), 1500)
    rel = np.linalg.norm(Y - V @ D) / np.linalg.norm(Y)
    assert rel < 1e-3, rel


def test_brute_force_tiny(orc):
    """Independent scalar transcription of the Lee-Seung updates on tiny inputs."""
    rng = np.random.default_rng(9)
    Np, Nk, K = 4, 3, 2
    Y = rng.uniform(-0.2, 1, size=(Np, Nk)).astype(np.float32)
    V = rng.uniform(0.2, 1, size=(Np, K)).tolist()
    D = rng.uniform(0.2, 1, size=(K, Nk)).tolist()
    V0 = np.array(V)
    D0 = np.array(D)
    y = [[max(float(Y[p][l]), 0.0) for l in range(Nk)] for p in range(Np)]
    for _ in range(3):
        newV = [[0.0] * K for _ in range(Np)]
        for p in range(Np):
            for k in range(K):
                num = sum(y[p][l] * D[k][l] for l in range(Nk))
                den = sum(V[p][j] * sum(D[j][l] * D[k][l] for l in range(Nk)) for j in range(K))
                newV[p][k] = V[p][k] * num / max(den, 1e-30)
        V = newV
        newD = [[0.0] * Nk for _ in range(K)]
        for k in range(K):
            for l in range(Nk):
                num = sum(V[p][k] * y[p][l] for p in range(Np))
                den = sum(sum(V[p][k] * V[p][j] for p in range(Np)) * D[j][l] for j in range(K))
                newD[k][l] = D[k][l] * num / max(den, 1e-30)
        D = newD
    Vo, Do = orc.nmf(Y, V0, D0, 3)
    np.testing.assert_allclose(Vo, V, rtol=1e-13)
    np.testing.assert_allclose(Do, D, rtol=1e-13)


def test_sampled_steps_match_full_iteration(orc):
    """oracle_nmf_vstep_rows / dstep_cols (used at full size) equal one full iteration."""
    pr = sd.make_problem(sd.custom(Nc=16, Nv=12, Nk=30, K=3, M=3))
    Y, V0, D0 = pr["Y"].numpy(), pr["V0"].numpy().astype(np.float64), pr["D0"].numpy().astype(np.float64)
    V1, D1 = orc.nmf(Y, V0, D0, 1)
    rows = np.array([0, 5, 17, Y.shape[0] - 1])
    cols = np.array([0, 3, 29])
    np.testing.assert_allclose(orc.nmf_vstep_rows(Y, V0, D0, rows), V1[rows], rtol=1e-13)
    np.testing.assert_allclose(orc.nmf_dstep_cols(Y, V1, D0, cols), D1[:, cols], rtol=1e-13)


def test_zero_iterations_is_identity(orc):
    Y = np.ones((3, 2), dtype=np.float32)
    V0 = np.full((3, 1), 0.5)
    D0 = np.full((1, 2), 0.25)
    V, D = orc.nmf(Y, V0, D0, 0)
    np.testing.assert_array_equal(V, V0)
    np.testing.assert_array_equal(D, D0)
