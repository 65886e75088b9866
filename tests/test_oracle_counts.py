"""Pins of oracle.counts_to_projections (NEXT-1: Eq. 2, with the Appendix-A
offset b_{v,k}, and the 1/2-count floor of DESIGN.md R7), CPU only.

* Closed forms: p = ln(y0 / y) for y, y0 >= 1 (computed here as the log of the ratio); y = 0
  uses the floor, p = ln(2 y0); y = y0 gives p = -b exactly.
* Indexing: y0 follows (r, c) = p mod N_r N_c and is shared by every view; b follows the view
  v = p div N_r N_c and the bin -- structured inputs where every element has a distinct value.
* Eq. 2 inverts Eq. 10: for integer counts drawn as y = y0 e^{-p} exactly (p = ln(y0 / y) by
  construction) the oracle returns that p.
* The generator's uint8 path (synthdata.make_problem(return_counts=True)) is fp32 of this
  function (R7, SURVEY §8(c) data-generator pin).
"""
import math

import numpy as np
import pytest

import oracle
import synthdata as sd


def test_closed_forms():
    y0 = np.array([[100, 100, 7, 0, 255, 1]], dtype=np.uint8)
    y = np.array([[50, 0, 7, 0, 1, 255]], dtype=np.uint8)
    P = oracle.counts_to_projections(y, y0, Nv=1)
    assert P[0, 0] == pytest.approx(math.log(2.0), rel=1e-15)
    assert P[0, 1] == pytest.approx(math.log(200.0), rel=1e-15)
    assert P[0, 2] == 0.0
    assert P[0, 3] == 0.0
    assert P[0, 4] == pytest.approx(math.log(255.0), rel=1e-15)
    assert P[0, 5] == pytest.approx(-math.log(255.0), rel=1e-15)
    b = np.array([[0.25, -1.5, 3.0, 0.0, 1e-3, -2.0]])
    Pb = oracle.counts_to_projections(y, y0, Nv=1, b=b)
    np.testing.assert_allclose(Pb, P - b, rtol=0, atol=1e-15)
    eq = oracle.counts_to_projections(y0, y0, Nv=1, b=b)
    assert np.array_equal(eq, -b)


def test_indexing_of_open_beam_and_offset():
    Nv, Nr, Nc, Nk = 3, 2, 4, 5
    rng = np.random.default_rng(0)
    y0 = rng.integers(1, 256, size=(Nr * Nc, Nk), dtype=np.uint8)
    y = rng.integers(1, 256, size=(Nv * Nr * Nc, Nk), dtype=np.uint8)
    b = rng.standard_normal((Nv, Nk))
    P = oracle.counts_to_projections(y, y0, Nv, b)
    for v in range(Nv):
        for r in range(Nr):
            for c in range(Nc):
                p = (v * Nr + r) * Nc + c
                for k in range(Nk):
                    want = math.log(float(y0[r * Nc + c, k]) / float(y[p, k])) - b[v, k]
                    assert P[p, k] == pytest.approx(want, rel=1e-12, abs=1e-13)


def test_inverts_eq10():
    # y = y0 exp(-p) with integer counts: choose y0 and y, p is then ln(y0 / y) exactly
    y0 = np.array([[200, 128, 90, 3]], dtype=np.uint8)
    p_true = np.array([[math.log(200 / 25), math.log(2.0), math.log(90 / 45), 0.0]])
    y = np.rint(y0 * np.exp(-p_true)).astype(np.uint8)
    assert list(y[0]) == [25, 64, 45, 3]
    np.testing.assert_allclose(oracle.counts_to_projections(y, y0, 1), p_true, rtol=0, atol=1e-14)


def test_generator_uint8_path_is_fp32_of_the_oracle():
    cfg = sd.custom(idx=31, Nc=16, Nv=6, Nr=2, Nk=40, K=3, M=3, counts=20.0)
    pr = sd.make_problem(cfg, return_counts=True)
    P = oracle.counts_to_projections(pr["y"].numpy(), pr["y0"].numpy(), cfg.Nv)
    assert np.array_equal(pr["Y"].numpy(), P.astype(np.float32))
