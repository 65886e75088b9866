"""GPU parity of the FMD back half (NEXT-2: Algorithm 2) through the
C ABI against the fp64 oracle: transformation matrix (Eq. 7), per-voxel NNLS material
estimation (Eq. 8), mu-spectra (Eq. 9), the Appendix-B identity, and the error paths."""
import numpy as np
import pytest
import torch

import oracle
import synthdata as sd

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def rel(a, b):
    a = a.detach().cpu().double().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, np.float64)
    b = b.detach().cpu().double().numpy() if isinstance(b, torch.Tensor) else np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def hs(cfg):
    from paper_2410_22500_b200 import Hsnct
    return Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)


@pytest.mark.parametrize("cfg,n_iter", [(sd.CONFIGS[1], 100), (sd.CONFIGS[2], 40)])
def test_fmd_pipeline_parity(cfg, n_iter):
    """decompose -> fbp -> FMD on the phantom's pure-material regions, vs the oracle on the
    same X and D."""
    pr = sd.make_problem(cfg)
    h = hs(cfg)
    V, D = pr["V0"].to(DEV).clone(), pr["D0"].to(DEV).clone()
    h.subspace_decompose(pr["Y"].to(DEV), V, D, n_iter)
    X = h.fbp(V)
    lab = torch.as_tensor(sd.region_labels(pr)).to(DEV).contiguous()
    nm = cfg.M if cfg.M <= cfg.K else cfg.K
    T = h.fmd_transform(X, lab, nm)
    Xm = h.fmd_materials(X, T)
    Dm = h.fmd_spectra(D, T)
    h.sync()
    Xn, Dn = X.cpu().numpy(), D.cpu().numpy()
    To, cnt = oracle.fmd_transform(Xn, sd.region_labels(pr), nm)
    assert cnt.min() > 0
    assert rel(T, To) <= 1e-5, rel(T, To)
    Xmo = oracle.fmd_materials(Xn, T.cpu().numpy())     # Eq. 8 on the GPU's T
    assert rel(Xm, Xmo) <= 1e-4, rel(Xm, Xmo)
    assert float(Xm.min()) >= 0.0
    Dmo = oracle.fmd_spectra(Dn, T.cpu().numpy())
    assert rel(Dm, Dmo) <= 1e-5, rel(Dm, Dmo)


def test_fmd_exact_mixtures_and_appendix_b():
    """x^s = x^m T exactly (pure regions + mixtures): T, x^m recovered; x^s (D^s)^T equals
    x^m (D^m)^T (Appendix B)."""
    cfg = sd.custom(idx=30, Nc=32, Nv=8, Nr=2, Nk=50, K=6, M=3)
    g = np.random.default_rng(5)
    Nm, K = 3, 6
    T = (g.random((Nm, K)) + 0.2).astype(np.float64)
    Nx = cfg.Nx
    xm = np.zeros((Nm, Nx))
    lab = np.full(Nx, -1, np.int32)
    for n in range(Nx):
        kind = n % 5
        if kind < Nm:
            xm[kind, n] = 1.0
            lab[n] = kind
        elif kind == Nm:
            xm[:, n] = g.random(Nm) * (g.random(Nm) > 0.3)
    X = (T.T @ xm).astype(np.float32)
    Tf = T.astype(np.float32)
    h = hs(cfg)
    Xd = torch.as_tensor(X).reshape(K, cfg.Nr, cfg.Nc, cfg.Nc).to(DEV).contiguous()
    labd = torch.as_tensor(lab).to(DEV)
    Tg = h.fmd_transform(Xd, labd, Nm)
    Xm = h.fmd_materials(Xd, Tg)
    D = torch.as_tensor(g.random((K, cfg.Nk)), dtype=torch.float32).to(DEV)
    Dm = h.fmd_spectra(D, Tg)
    h.sync()
    assert rel(Tg, Tf) <= 1e-6
    assert rel(Xm.reshape(Nm, -1), xm) <= 1e-5, rel(Xm.reshape(Nm, -1), xm)
    lhs = Xd.reshape(K, -1).T.double() @ D.double()
    rhs = Xm.reshape(Nm, -1).T.double() @ Dm.double()
    assert rel(rhs, lhs) <= 1e-5


def test_fmd_errors():
    from paper_2410_22500_b200 import HsnctError
    cfg = sd.custom(idx=31, Nc=16, Nv=8, Nr=1, Nk=20, K=3, M=2)
    h = hs(cfg)
    X = torch.rand((3, 1, 16, 16), device=DEV)
    lab = torch.zeros(256, dtype=torch.int32, device=DEV)
    with pytest.raises(HsnctError):            # n_mat > K
        h.fmd_transform(X, lab, 4)
    h.fmd_transform(X, lab, 2)                  # region 1 is empty -> deferred data error
    with pytest.raises(HsnctError) as e:
        h.sync()
    assert e.value.status == 2 and "region is empty" in str(e.value)
    lab[0] = 5                                  # label >= n_mat -> deferred data error
    lab[1] = 1
    h.fmd_transform(X, lab, 2)
    with pytest.raises(HsnctError) as e:
        h.sync()
    assert e.value.status == 2 and "label outside" in str(e.value)
    lab[0] = -3                                 # labels < -1 are not "none": data error
    h.fmd_transform(X, lab, 2)
    with pytest.raises(HsnctError) as e:
        h.sync()
    assert e.value.status == 2 and "label outside" in str(e.value)


def test_fmd_nnls_random_supports():
    """Eq. 8 on random mixed-sign x^s with N_m = K = 6: solutions of every support size (the
    Lawson-Hanson front end and its enumeration fallback), vs the oracle's NNLS."""
    cfg = sd.custom(idx=31, Nc=48, Nv=8, Nr=2, Nk=12, K=6, M=6)
    g = np.random.default_rng(11)
    K = Nm = 6
    T = (np.eye(Nm, K) + 0.3 * g.random((Nm, K))).astype(np.float32)
    X = g.standard_normal((K, cfg.Nx)).astype(np.float32)
    h = hs(cfg)
    Xd = torch.as_tensor(X).reshape(K, cfg.Nr, cfg.Nc, cfg.Nc).to(DEV).contiguous()
    Xm = h.fmd_materials(Xd, torch.as_tensor(T).to(DEV))
    h.sync()
    Xmo = oracle.fmd_materials(X.reshape(K, cfg.Nr, cfg.Nc, cfg.Nc), T)
    a = Xm.reshape(Nm, -1).cpu().double().numpy()
    b = np.asarray(Xmo, np.float64).reshape(Nm, -1)
    assert rel(a, b) <= 1e-5, rel(a, b)
    assert np.abs(a - b).max() <= 1e-4 * max(1.0, np.abs(b).max())
    supp = (b > 0).sum(axis=0)
    assert set(np.unique(supp)) >= {0, 1, 2, 3, 4}  # the data really exercise many support sizes
