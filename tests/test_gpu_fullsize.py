"""GPU parity at BASELINE.json's full sizes (C3, C4, C5), in the launch configuration
bench.py times, on sampled outputs the oracle computes one by one:

* one Lee-Seung iteration from the seeded init: V_1 on sampled rows (oracle V half-step on
  those rows of Y+ with V_0, D_0) and D_1 on sampled bins (oracle D half-step on those bins
  with the GPU's V_1 and D_0);
* a later iteration inside one persistent launch: decompose(2) from (V_1, D_1) must equal,
  within fp32 summation order, decompose(1) twice (each single step is oracle-checked above);
* FBP of the K subspace sinograms on sampled slices (oracle FBP of those slices);
* synthesis on a sampled window and DHR on a sampled slice x bin window.
Tolerances as in test_gpu_parity.py (one step: 1e-4; FBP / synthesis / DHR: 1e-4).
"""
import gc

import numpy as np
import pytest
import torch

import oracle
import synthdata as sd

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def sample_rows(Np, n, seed):
    g = np.random.default_rng(seed)
    r = np.concatenate([[0, 1, 2, 3, Np - 4, Np - 3, Np - 2, Np - 1], g.integers(0, Np, n)])
    return np.unique(r)


@pytest.mark.parametrize("ci", [3, 4, 5])
def test_fullsize_sampled_parity(ci):
    from paper_2410_22500_b200 import Hsnct
    cfg = sd.CONFIGS[ci]
    free, _ = torch.cuda.mem_get_info()
    need = 2.2 * 4 * cfg.Np * cfg.Nk + 6 * cfg.K * cfg.Nx * 4
    if free < need:
        pytest.skip(f"needs {need / 1e9:.0f} GB of free device memory, {free / 1e9:.0f} GB free")
    pr = sd.make_problem(cfg, device=DEV)
    Y, V0, D0 = pr["Y"], pr["V0"], pr["D0"]
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    try:
        # ---- one iteration from the init
        V1, D1 = V0.clone(), D0.clone()
        h.subspace_decompose(Y, V1, D1, 1)
        h.sync()
        rows = sample_rows(cfg.Np, 384, 1000 * ci + 11)
        ri = torch.as_tensor(rows, device=DEV)
        Vexp = oracle.nmf_vstep_rows(Y[ri].cpu().numpy(), V0[ri].cpu().numpy(), D0.cpu().numpy(),
                                     np.arange(rows.size))
        assert rel(V1[ri].cpu().numpy(), Vexp) <= 1e-4, rel(V1[ri].cpu().numpy(), Vexp)
        cols = np.unique(np.concatenate([[0, cfg.Nk - 1], np.random.default_rng(ci).integers(0, cfg.Nk, 10)]))
        ci_t = torch.as_tensor(cols, device=DEV)
        Dexp = oracle.nmf_dstep_cols(Y[:, ci_t].contiguous().cpu().numpy(), V1.cpu().numpy(),
                                     D0[:, ci_t].cpu().numpy(), np.arange(cols.size))
        assert rel(D1[:, ci_t].cpu().numpy(), Dexp) <= 1e-4, rel(D1[:, ci_t].cpu().numpy(), Dexp)
        # ---- iterations 2..3 inside one launch vs two single launches
        V3, D3 = V1.clone(), D1.clone()
        h.subspace_decompose(Y, V3, D3, 2)
        Va, Da = V1.clone(), D1.clone()
        h.subspace_decompose(Y, Va, Da, 1)
        h.subspace_decompose(Y, Va, Da, 1)
        h.sync()
        assert rel(V3.cpu().numpy(), Va.cpu().numpy()) <= 1e-5
        assert rel(D3.cpu().numpy(), Da.cpu().numpy()) <= 1e-5
        # ---- FBP on sampled slices
        X = h.fbp(V3)
        h.sync()
        sl = sorted({0, cfg.Nr // 2, cfg.Nr - 1})
        Vr = V3.reshape(cfg.Nv, cfg.Nr, cfg.Nc, cfg.K)
        for r in sl:
            Xo = oracle.fbp(Vr[:, r].reshape(-1, cfg.K).cpu().numpy(), cfg.Nv, 1, cfg.Nc)
            assert rel(X[:, r].cpu().numpy(), Xo.reshape(cfg.K, cfg.Nc, cfg.Nc)) <= 1e-4
        # ---- synthesis on a window (one slice, a ragged bin range)
        r = cfg.Nr // 3
        b0, nb = 5, cfg.Nk - 11
        Xh = h.synthesize(X, D3, r, 1, b0, nb)
        h.sync()
        Xho = oracle.synthesize(X[:, r:r + 1].cpu().numpy(), D3.cpu().numpy()[:, b0:b0 + nb])
        assert rel(Xh.cpu().numpy(), Xho) <= 1e-4
        # ---- FMD back half: T from seeded random regions (oracle on the full X), NNLS on
        #      sampled voxels (oracle with the GPU's T), spectra
        nm = min(cfg.M, cfg.K)
        lab = torch.as_tensor(np.random.default_rng(ci).integers(-1, nm, cfg.Nx), dtype=torch.int32).to(DEV)
        T = h.fmd_transform(X, lab, nm)
        Xm = h.fmd_materials(X, T)
        Dm = h.fmd_spectra(D3, T)
        h.sync()
        Xh_ = X.reshape(cfg.K, -1)
        To, _ = oracle.fmd_transform(Xh_.cpu().numpy(), lab.cpu().numpy(), nm)
        assert rel(T.cpu().numpy(), To) <= 1e-5
        vox = torch.as_tensor(sample_rows(cfg.Nx, 2000, ci), device=DEV)
        Xmo = oracle.fmd_materials(Xh_[:, vox].cpu().numpy(), T.cpu().numpy())
        assert rel(Xm.reshape(nm, -1)[:, vox].cpu().numpy(), Xmo) <= 1e-4
        assert rel(Dm.cpu().numpy(), oracle.fmd_spectra(D3.cpu().numpy(), T.cpu().numpy())) <= 1e-5
        del Xh_, Xm, lab
        # ---- DHR on one slice x 8 bins
        Xd = h.dhr(Y, r, 1, 100, 8)
        h.sync()
        Yr = Y.reshape(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk)[:, r, :, 100:108].reshape(-1, 8).contiguous()
        Xdo = oracle.dhr(Yr.cpu().numpy(), cfg.Nv, 1, cfg.Nc)
        assert rel(Xd.cpu().numpy(), Xdo) <= 1e-4
    finally:
        h.close()
        del pr, Y, V0, D0
        gc.collect()
        torch.cuda.empty_cache()
