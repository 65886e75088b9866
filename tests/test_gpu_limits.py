"""GPU parity at the boundary's size limits (include/hsnct.h: 2 <= N_c <= 1024,
K * round_up(N_k, 4) <= 51200, K <= 16) and at the degenerate end (N_c = 2, N_k = 1, K = 1),
against the fp64 oracle.  Tolerances as tests/test_gpu_parity.py (north_star): FBP and
synthesis <= 1e-4 relative L2, NMF <= 1e-3 on V, D and x^h.
"""
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


def handle(cfg):
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2410_22500_b200 import Hsnct
    return Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)


def padded(Y):
    """Y on the device in rows of ld = round_up(N_k, 4) floats (the boundary's ld rule), the
    padding NaN-poisoned (must be ignored)."""
    Np, Nk = Y.shape
    buf = torch.full((Np, (Nk + 3) // 4 * 4), float("nan"), dtype=torch.float32, device=DEV)
    buf[:, :Nk] = Y.to(DEV)
    return buf[:, :Nk]


def pipeline(cfg, n_iter):
    pr = sd.make_problem(cfg)
    h = handle(cfg)
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    h.subspace_decompose(padded(pr["Y"]), V, D, n_iter)
    X = h.fbp(V)
    Xh = h.synthesize(X, D)
    h.sync()
    Vo, Do = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), n_iter)
    return pr, h, V, D, X, Xh, Vo, Do


def test_max_detector_width_nc1024():
    """N_c = 1024 (FFT length P = 2048: the shared-memory radix-2 ramp filter, and the KC = 8
    DHR backprojection) through the whole path, and FBP of the oracle's own V."""
    cfg = sd.custom(idx=91, Nc=1024, Nv=6, Nr=1, Nk=8, K=2, M=2)
    pr, h, V, D, X, Xh, Vo, Do = pipeline(cfg, 10)
    assert rel(V, Vo) <= 1e-3 and rel(D, Do) <= 1e-3, (rel(V, Vo), rel(D, Do))
    Xo = oracle.fbp(Vo, cfg.Nv, cfg.Nr, cfg.Nc)
    assert rel(Xh, oracle.synthesize(Xo, Do)) <= 1e-3
    # the FBP stage alone on identical input (the oracle's V)
    Xg = h.fbp(torch.as_tensor(Vo, dtype=torch.float32, device=DEV))
    h.sync()
    assert rel(Xg, Xo) <= 1e-4, rel(Xg, Xo)
    # DHR of two bins at this width
    Xd = h.dhr(pr["Y"].to(DEV), bin0=3, n_bins=2)
    h.sync()
    Xdo = oracle.dhr(pr["Y"].numpy(), cfg.Nv, cfg.Nr, cfg.Nc, bin0=3, n_bins=2)
    assert rel(Xd, Xdo) <= 1e-4, rel(Xd, Xdo)


def test_max_subspace_times_bins():
    """K = 16 with K * round_up(N_k, 4) = 51200 exactly (the largest D tile the boundary accepts;
    few rows, so the plan takes the fallback kernels)."""
    cfg = sd.custom(idx=92, Nc=8, Nv=4, Nr=1, Nk=3200, K=16, M=4)
    pr = sd.make_problem(cfg)
    h = handle(cfg)
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    obj = torch.zeros(2 * 6, dtype=torch.float64, device=DEV)
    h.subspace_decompose(pr["Y"].to(DEV), V, D, 6, obj_trace=obj)
    h.sync()
    Vo, Do, objo = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), 6, objective=True)
    assert rel(V, Vo) <= 1e-3 and rel(D, Do) <= 1e-3, (rel(V, Vo), rel(D, Do))
    np.testing.assert_allclose(obj.cpu().numpy(), objo, rtol=1e-3)


def test_smallest_geometry():
    """N_c = 2, N_v = 2, N_k = 1, K = 1: every stage on the degenerate shape."""
    cfg = sd.custom(idx=93, Nc=2, Nv=2, Nr=1, Nk=1, K=1, M=1)
    pr, h, V, D, X, Xh, Vo, Do = pipeline(cfg, 5)
    assert rel(V, Vo) <= 1e-3 and rel(D, Do) <= 1e-3, (rel(V, Vo), rel(D, Do))
    Xo = oracle.fbp(Vo, cfg.Nv, cfg.Nr, cfg.Nc)
    assert rel(Xh, oracle.synthesize(Xo, Do)) <= 1e-3
