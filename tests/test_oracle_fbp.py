"""Pins for the oracle's FBP pieces (oracle.c: ramp filter, backprojection, fbp,
synthesis, dhr) against closed forms, analytic phantoms, the adjoint identity
and the FBP/DHR linearity identity (
DESIGN.md R10-R17)."""
import math

import numpy as np
import pytest
import torch

import synthdata as sd


# ---------------------------------------------------------------- ramp filter
def test_ramp_kernel_values(orc):
    assert orc.ramp_kernel(0) == 0.25
    for d in (2, -2, 4, 100):
        assert orc.ramp_kernel(d) == 0.0
    for d in (1, -1, 3, -7):
        assert orc.ramp_kernel(d) == pytest.approx(-1.0 / (math.pi ** 2 * d * d), rel=1e-15)


def test_ramp_filter_frequency_response(orc):
    """The Kak-Slaney kernel is the sampled band-limited ramp: its DTFT is |f|
    for |f| <= 1/2.  A long cosine of frequency f comes out scaled by |f| away
    from the ends (truncation error O(1/(pi^2 N)))."""
    N = 4096
    m = np.arange(N)
    for f in (0.05, 0.125, 0.3):
        s = np.cos(2 * math.pi * f * m + 0.3)
        q = orc.ramp_filter_rows(s[None, :])[0]
        mid = slice(N // 2 - 200, N // 2 + 200)
        np.testing.assert_allclose(q[mid], f * s[mid], atol=2e-4)


def test_ramp_filter_impulse_and_linearity(orc):
    Nc = 33
    s = np.zeros((2, Nc))
    s[0, 10] = 1.0
    s[1] = np.linspace(-1, 1, Nc)
    q = orc.ramp_filter_rows(s)
    np.testing.assert_allclose(q[0], [orc.ramp_kernel(c - 10) for c in range(Nc)], rtol=1e-15)
    q2 = orc.ramp_filter_rows(2.0 * s[0:1] - 3.0 * s[1:2])
    np.testing.assert_allclose(q2[0], 2 * q[0] - 3 * q[1], atol=1e-14)


def test_ramp_dc_gain_tail(orc):
    """sum_d h[d] over |d| <= Nc-1 = (2/pi^2) sum_{odd d >= Nc} 1/d^2 since the
    full sum is 1/4 - (2/pi^2)(pi^2/8) = 0; the tail is ~ 1/(pi^2 (Nc-1))."""
    for Nc in (64, 256, 512):
        q = orc.ramp_filter_rows(np.ones((1, 2 * Nc - 1)))[0]
        dc = q[Nc - 1]   # centre sample sees |d| <= Nc-1 on both sides
        L = 200001  # remainder sum_{odd d >= L} 1/d^2 = 1/(2(L-1)) + O(L^-3)
        tail = sum(1.0 / d ** 2 for d in range(Nc + (Nc % 2 == 0), L, 2)) + 1.0 / (2 * (L - 1))
        assert dc == pytest.approx(2.0 / math.pi ** 2 * tail, rel=1e-4)


# -------------------------------------------------------------- backprojection
def test_single_view_impulse_theta0(orc):
    Nv, Nc, c0 = 8, 17, 5
    Q = np.zeros((Nv, Nc))
    Q[0, c0] = 1.0
    X = orc.backproject_slice(Q)
    expect = np.zeros((Nc, Nc))
    expect[:, c0] = math.pi / Nv
    np.testing.assert_allclose(X, expect, atol=1e-15)


def test_single_view_impulse_theta90(orc):
    Nv, Nc, c0 = 8, 17, 12
    Q = np.zeros((Nv, Nc))
    Q[Nv // 2, c0] = 1.0
    X = orc.backproject_slice(Q)
    expect = np.zeros((Nc, Nc))
    expect[c0, :] = math.pi / Nv
    np.testing.assert_allclose(X, expect, atol=1e-12)


def test_adjoint_identity(orc):
    rng = np.random.default_rng(1)
    for Nv, Nc in ((8, 32), (7, 21), (12, 16)):
        x = rng.normal(size=(Nc, Nc))
        y = rng.normal(size=(Nv, Nc))
        lhs = np.sum(orc.splat_project_slice(x, Nv) * y)
        rhs = np.sum(x * orc.backproject_slice(y))
        assert lhs == pytest.approx(rhs, rel=1e-12)


def test_custom_angles_match_default(orc):
    rng = np.random.default_rng(4)
    Q = rng.normal(size=(9, 20))
    a = np.arange(9) * math.pi / 9
    np.testing.assert_allclose(orc.backproject_slice(Q, a), orc.backproject_slice(Q), rtol=1e-15)


# ------------------------------------------------------------ analytic phantoms
def _disk_sino(Nv, Nc, rho, mu=1.0, x0=0.0, y0=0.0, a=None, b=None, alpha=0.0):
    th = torch.as_tensor(sd.view_angles(Nv), dtype=torch.float64)[:, None]
    t = (torch.arange(Nc, dtype=torch.float64) - 0.5 * (Nc - 1))[None, :]
    return sd.ellipse_line_integrals(th, t, x0, y0, a or rho, b or rho, alpha, mu).numpy()


@pytest.mark.parametrize("Nc,Nv", [(64, 90), (256, 180)])
def test_fbp_analytic_disk_interior(orc, Nc, Nv):
    rho = 0.3 * Nc
    P = _disk_sino(Nv, Nc, rho)
    V = P.reshape(Nv * Nc, 1)  # Nr = 1, K = 1
    X = orc.fbp(V, Nv, 1, Nc)[0, 0]
    half = 0.5 * (Nc - 1)
    yy, xx = np.mgrid[0:Nc, 0:Nc] - half
    inner = np.hypot(xx, yy) < 0.8 * rho
    outer = np.hypot(xx, yy) > 1.2 * rho
    assert X[inner].mean() == pytest.approx(1.0, abs=3e-3)
    assert abs(X[outer].mean()) < 2e-2


def test_fbp_analytic_offcentre_ellipse(orc):
    Nc, Nv = 128, 120
    P = _disk_sino(Nv, Nc, None, mu=2.0, x0=15.0, y0=-10.0, a=25.0, b=14.0, alpha=0.6)
    X = orc.fbp(P.reshape(-1, 1), Nv, 1, Nc)[0, 0]
    half = 0.5 * (Nc - 1)
    yy, xx = np.mgrid[0:Nc, 0:Nc] - half
    ca, sa = math.cos(0.6), math.sin(0.6)
    xr = (xx - 15.0) * ca + (yy + 10.0) * sa
    yr = -(xx - 15.0) * sa + (yy + 10.0) * ca
    inner = (xr / 20.0) ** 2 + (yr / 10.0) ** 2 <= 1
    assert X[inner].mean() == pytest.approx(2.0, abs=1e-2)


def test_analytic_chord_vs_naive_radon(orc):
    """The generator's analytic line integral vs a naive ray-sampled Radon of a
    supersampled rasterised disk (SPEC test idea: chord = 2 rho mu within 2%)."""
    cfg = sd.custom(Nc=64, Nv=16, M=1)
    shp = [sd.Ellipsoid(0, 3.0, -2.0, 0.0, 18.0, 11.0, math.inf, 0.4)]
    img = sd.rasterize(shp, cfg, 0, supersample=8)[0]
    Pn = orc.radon_naive(img, 16, step=0.25)
    Pa = sd.material_sinograms(shp, cfg)[0, :, 0, :].numpy()
    # away from the silhouette edges (where the rasterised boundary is blurred
    # by +-1 px) the two agree to 2 % of the peak; the per-view mass matches the area
    interior = (np.roll(Pa, 2, axis=1) > 0) & (np.roll(Pa, -2, axis=1) > 0)
    assert np.abs(Pn - Pa)[interior].max() < 0.02 * Pa.max()
    np.testing.assert_allclose(Pn.sum(1), math.pi * 18.0 * 11.0, rtol=5e-3)
    # centred disk: central bin = 2 rho mu
    P0 = _disk_sino(4, 65, 20.0)
    np.testing.assert_allclose(P0[:, 32], 40.0, rtol=1e-14)


def test_centred_disk_rotation_symmetry(orc):
    Nc, Nv = 48, 32
    P = _disk_sino(Nv, Nc, 15.0)
    X = orc.fbp(P.reshape(-1, 1), Nv, 1, Nc)[0, 0]
    np.testing.assert_allclose(np.rot90(X), X, atol=1e-12)


def test_fbp_zero_and_linearity(orc):
    rng = np.random.default_rng(8)
    Nv, Nr, Nc, K = 6, 2, 12, 2
    V = rng.normal(size=(Nv * Nr * Nc, K))
    X = orc.fbp(V, Nv, Nr, Nc)
    assert np.all(orc.fbp(np.zeros_like(V), Nv, Nr, Nc) == 0)
    X2 = orc.fbp(2 * V[:, ::-1], Nv, Nr, Nc)
    np.testing.assert_allclose(X2, 2 * X[::-1], atol=1e-13)


def test_fbp_slices_decouple(orc):
    """Parallel beam: slice r of X depends only on detector row r."""
    rng = np.random.default_rng(3)
    Nv, Nr, Nc = 5, 3, 10
    V = rng.normal(size=(Nv * Nr * Nc, 1))
    X = orc.fbp(V, Nv, Nr, Nc)
    V1 = V.reshape(Nv, Nr, Nc)[:, 1, :].reshape(-1, 1)
    np.testing.assert_allclose(X[0, 1], orc.fbp(V1, Nv, 1, Nc)[0, 0], rtol=1e-14)


# ------------------------------------------------------------------ synthesis
def test_synthesize_identity_and_unit(orc):
    rng = np.random.default_rng(2)
    K, Nr, Nc = 5, 2, 4
    X = rng.normal(size=(K, Nr, Nc, Nc))
    Xh = orc.synthesize(X, np.eye(K))
    np.testing.assert_array_equal(Xh, X.reshape(K, -1).T)
    D = rng.normal(size=(K, 9))
    Xu = np.zeros_like(X)
    Xu[3, 1, 2, 1] = 1.0
    n = (1 * Nc + 2) * Nc + 1
    np.testing.assert_array_equal(orc.synthesize(Xu, D)[n], D[3])


def test_synthesize_matches_matmul_and_windows(orc):
    rng = np.random.default_rng(6)
    K, Nr, Nc, Nk = 3, 4, 5, 11
    X = rng.normal(size=(K, Nr, Nc, Nc))
    D = rng.normal(size=(K, Nk))
    full = X.reshape(K, -1).T @ D
    np.testing.assert_allclose(orc.synthesize(X, D), full, rtol=1e-13, atol=1e-14)
    w = orc.synthesize(X, D, slice0=1, n_slices=2, bin0=3, n_bins=5)
    np.testing.assert_allclose(w, full[Nc * Nc:3 * Nc * Nc, 3:8], rtol=1e-13, atol=1e-14)
    with pytest.raises(ValueError):
        orc.synthesize(X, D, slice0=3, n_slices=2)


# ------------------------------------------------------------------------- DHR
def test_dhr_bin_equals_fbp_of_that_bin(orc):
    rng = np.random.default_rng(12)
    Nv, Nr, Nc, Nk = 6, 2, 10, 7
    Y = rng.normal(size=(Nv * Nr * Nc, Nk)).astype(np.float32)
    Xh = orc.dhr(Y, Nv, Nr, Nc)
    for l in (0, 4, 6):
        X = orc.fbp(Y[:, l:l + 1].astype(np.float64), Nv, Nr, Nc)[0]
        np.testing.assert_allclose(Xh[:, l], X.reshape(-1), rtol=1e-14, atol=1e-15)


def test_linearity_identity_fhr_equals_dhr(orc):
    """FBP is linear, so for Y = V D exactly: sum_k FBP(V_k) D[k, l] = FBP(Y_l)
    (Eq. 6 after Algorithm 1's reconstruction step equals DHR)."""
    rng = np.random.default_rng(13)
    Nv, Nr, Nc, Nk, K = 10, 2, 16, 9, 3
    V = rng.integers(0, 8, size=(Nv * Nr * Nc, K)).astype(np.float64)
    D = rng.integers(0, 8, size=(K, Nk)).astype(np.float64) / 4.0
    Y = (V @ D).astype(np.float32)  # dyadic: exact in fp32
    assert np.array_equal(Y.astype(np.float64), V @ D)
    X = orc.fbp(V, Nv, Nr, Nc)
    lhs = orc.synthesize(X, D)
    rhs = orc.dhr(Y, Nv, Nr, Nc)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-11, atol=1e-11)
    w = orc.dhr(Y, Nv, Nr, Nc, slice0=1, n_slices=1, bin0=2, n_bins=4)
    np.testing.assert_allclose(w, rhs[Nc * Nc:, 2:6], rtol=1e-14)
