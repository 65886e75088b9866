"""GPU parity of the MBIR path (NEXT-3: Eq. 5; R24-R26) through the
C ABI against the fp64 oracle (oracle.mbir_project_slice, oracle.mbir_slice, oracle.mbir).

* hsnct_project = A on every (channel, slice): ragged N_c, N_c > 128 (several warps per view),
  K = 1 .. 10 (both projector instantiation families), custom angles with views exactly on the
  45-degree class boundary.
* hsnct_mbir after n SQS iterations vs the oracle, plus the objective trace (summed over
  channels and slices) and its monotonicity; p = 1, 1.2, 2 (p = 2: the u = 1 branch).
* n_iter = 0 leaves X unchanged and reports the x0 objective; argument errors are E_ARG.
* C5 geometry (512 x 512, 256 slices, 64 views, K = 6) in the bench's launch configuration,
  5 iterations, checked on sampled slices that the oracle runs one by one.

Tolerances (fp32 kernels vs fp64 oracle): projection rel-L2 1e-5 (sums of <= 3 N_c products of
weights in [0, 1]); MBIR rel-L2 2e-4 after <= 20 contractive SQS steps (each step's fp32
rounding ~1e-6 relative, fast lg2/ex2 in w(d) ~2e-7); objective rtol 1e-4.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synthdata as sd

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def rel(a, b):
    a = a.detach().cpu().double().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def make(Nv, Nr, Nc, K, angles=None):
    from paper_2410_22500_b200 import Hsnct
    return Hsnct(Nv, Nr, Nc, max(K, 4), K, angles=angles, device=0)


def phantom(K, Nr, Nc, seed):
    """Piecewise-constant discs per channel plus a little texture, >= 0."""
    rng = np.random.default_rng(seed)
    X = np.zeros((K, Nr, Nc, Nc))
    yy, xx = np.mgrid[0:Nc, 0:Nc] - 0.5 * (Nc - 1)
    for k in range(K):
        for r in range(Nr):
            for _ in range(4):
                cx, cy = rng.uniform(-0.3, 0.3, 2) * Nc
                rad = rng.uniform(0.08, 0.25) * Nc
                X[k, r][(xx - cx) ** 2 + (yy - cy) ** 2 < rad ** 2] += rng.uniform(0.2, 1.0)
    return X + 0.02 * rng.random(X.shape)


def project_oracle(X, Nv, angles=None):
    """A X for every (channel, slice) in the layout of V [Np, K]."""
    K, Nr, Nc, _ = X.shape
    P = np.zeros((Nv, Nr, Nc, K))
    for k in range(K):
        for r in range(Nr):
            P[:, r, :, k] = oracle.mbir_project_slice(X[k, r], Nv, angles=angles)
    return P.reshape(-1, K)


@pytest.mark.parametrize("Nv,Nr,Nc,K", [(20, 2, 37, 3), (12, 1, 130, 1), (9, 2, 200, 8), (7, 1, 64, 10),
                                        (5, 1, 16, 2), (3, 1, 300, 6)])
def test_project_parity(Nv, Nr, Nc, K):
    X = np.random.default_rng(Nc + K).random((K, Nr, Nc, Nc))
    h = make(Nv, Nr, Nc, K)
    P = h.project(torch.tensor(X, dtype=torch.float32, device=DEV))
    h.sync()
    e = rel(P, project_oracle(X, Nv))
    print(f"Nv={Nv} Nr={Nr} Nc={Nc} K={K}: rel-L2 {e:.2e}")
    assert e <= 1e-5, e
    h.close()


def test_project_custom_angles_class_boundary():
    Nc, K = 41, 2
    ang = np.array([0.0, math.pi / 4, 3 * math.pi / 4, math.pi / 2, 0.3, 2.0, 1.1, -0.7, 3.5])
    X = np.random.default_rng(2).random((K, 1, Nc, Nc))
    h = make(len(ang), 1, Nc, K, angles=ang)
    P = h.project(torch.tensor(X, dtype=torch.float32, device=DEV))
    h.sync()
    assert rel(P, project_oracle(X, len(ang), angles=ang)) <= 1e-5
    h.close()


def mbir_case(Nv, Nr, Nc, K, n_iter, prm, seed, angles=None):
    Xt = phantom(K, Nr, Nc, seed)
    rng = np.random.default_rng(seed + 1)
    Y = project_oracle(Xt, Nv, angles)
    Y = Y + 0.02 * np.abs(Y).mean() * rng.standard_normal(Y.shape)
    X0 = np.clip(Xt + 0.3 * rng.standard_normal(Xt.shape), 0, None)
    h = make(Nv, Nr, Nc, K, angles)
    V = torch.tensor(Y, dtype=torch.float32, device=DEV)
    X = torch.tensor(X0, dtype=torch.float32, device=DEV)
    obj = torch.zeros(n_iter + 1, dtype=torch.float64, device=DEV)
    h.mbir(V, X, n_iter, *prm, obj_trace=obj)
    h.sync()
    Xo = oracle.mbir(Y, Nv, Nr, Nc, X0, prm, n_iter, angles=angles)
    objo = np.zeros(n_iter + 1)
    Yr = Y.reshape(Nv, Nr, Nc, K)
    for k in range(K):
        for r in range(Nr):
            objo += oracle.mbir_slice(Yr[:, r, :, k], X0[k, r], prm, n_iter, angles=angles, objective=True)[1]
    h.close()
    return X, Xo, obj.cpu().numpy(), objo, X0


@pytest.mark.parametrize("Nv,Nr,Nc,K,p", [(24, 2, 48, 3, 1.2), (16, 1, 150, 6, 1.2), (10, 1, 40, 10, 1.2),
                                          (18, 1, 33, 2, 2.0), (18, 1, 33, 2, 1.0)])
def test_mbir_parity(Nv, Nr, Nc, K, p):
    n_iter = 20
    prm = oracle.mbir_params(2.0, 0.1, p=p)
    X, Xo, obj, objo, X0 = mbir_case(Nv, Nr, Nc, K, n_iter, prm, seed=Nc + K)
    e = rel(X, Xo)
    moved = rel(X0, Xo)
    print(f"Nv={Nv} Nc={Nc} K={K} p={p}: rel-L2 {e:.2e} (x0 -> x_n moved {moved:.2e}), "
          f"obj {objo[0]:.4e} -> {objo[-1]:.4e}")
    assert moved > 1e-2            # the iteration did something
    assert e <= 2e-4, e
    np.testing.assert_allclose(obj, objo, rtol=1e-4)
    assert np.all(np.diff(obj) <= 1e-5 * np.abs(obj[:-1])), "objective increased"
    assert float(X.min()) >= 0.0


def test_mbir_custom_angles():
    ang = np.sort(np.random.default_rng(9).uniform(0, math.pi, 15))
    prm = oracle.mbir_params(1.0, 0.2, p=1.1, T=2.0)
    X, Xo, obj, objo, _ = mbir_case(15, 1, 35, 2, 10, prm, seed=5, angles=ang)
    assert rel(X, Xo) <= 2e-4
    np.testing.assert_allclose(obj, objo, rtol=1e-4)


def test_mbir_zero_iterations_and_errors():
    from paper_2410_22500_b200 import HsnctError
    Nv, Nr, Nc, K = 8, 1, 20, 2
    h = make(Nv, Nr, Nc, K)
    rng = np.random.default_rng(1)
    X0 = torch.tensor(rng.random((K, Nr, Nc, Nc)), dtype=torch.float32, device=DEV)
    V = torch.tensor(rng.random((Nv * Nr * Nc, K)), dtype=torch.float32, device=DEV)
    X = X0.clone()
    obj = torch.zeros(1, dtype=torch.float64, device=DEV)
    h.mbir(V, X, 0, 1.0, 0.5, obj_trace=obj)
    h.sync()
    assert torch.equal(X, X0)
    prm = oracle.mbir_params(1.0, 0.5)
    o = sum(oracle.mbir_slice(V.cpu().double().numpy().reshape(Nv, Nr, Nc, K)[:, 0, :, k],
                              X0[k, 0].cpu().double().numpy(), prm, 0, objective=True)[1][0] for k in range(K))
    assert float(obj[0]) == pytest.approx(o, rel=1e-5)
    for bad in [dict(q=1.5), dict(p=0.5), dict(p=2.5), dict(sigma_v=0.0), dict(sigma_x=-1.0), dict(T=0.0),
                dict(sigma_v=float("nan"))]:
        kw = dict(sigma_v=1.0, sigma_x=0.5, p=1.2, q=2.0, T=1.0)
        kw.update(bad)
        with pytest.raises(HsnctError):
            h.mbir(V, X, 2, **kw)
    with pytest.raises(HsnctError):
        h.mbir(V, X, -1, 1.0, 0.5)
    h.close()


@pytest.mark.slow
def test_mbir_c5_sampled_slices():
    """C5 geometry, the launch configuration the bench times; 5 iterations from the FBP of
    synthetic subspace sinograms; slices 0, 128, 255 checked against the oracle."""
    cfg = sd.CONFIGS[5]
    n_iter = 5
    from paper_2410_22500_b200 import Hsnct
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    g = torch.Generator(device="cpu").manual_seed(3)
    Xt = torch.rand((cfg.K, 1, cfg.Nc, cfg.Nc), generator=g, dtype=torch.float64)
    Pt = project_oracle(Xt.numpy(), cfg.Nv)                      # one slice's sinogram
    Vs = torch.tensor(Pt, dtype=torch.float32).reshape(cfg.Nv, 1, cfg.Nc, cfg.K)
    scale = torch.linspace(0.5, 1.5, cfg.Nr, dtype=torch.float32).reshape(1, cfg.Nr, 1, 1)
    V = (Vs * scale).reshape(-1, cfg.K).contiguous().to(DEV)      # slice r = (0.5 + r/255) * slice 0
    X = h.fbp(V).clamp_(min=0)
    X0 = X.clone()
    prm = oracle.mbir_params(5.0, 0.05)
    h.mbir(V, X, n_iter, *prm)
    h.sync()
    Vc = V.cpu().double().numpy().reshape(cfg.Nv, cfg.Nr, cfg.Nc, cfg.K)
    for r in (0, 128, cfg.Nr - 1):
        for k in range(cfg.K):
            xo = oracle.mbir_slice(Vc[:, r, :, k], X0[k, r].cpu().double().numpy(), prm, n_iter)
            e = rel(X[k, r], xo)
            assert e <= 2e-4, (r, k, e)
    h.close()
