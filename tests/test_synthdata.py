"""Pins of the seeded input generator (SURVEY.md §8(c) "Data-gen"), CPU only.

* With noise disabled (real-valued counts), Eq. 2 inverts Eq. 10
   exactly: -log(C e^{-p} / C) = p to 1e-12 (fp64).
* The 256-entry log table is ln(max(n, 1/2)) (reading R7) and the integer-count path builds
  Y = fp32(L[y0] - L[y]) elementwise, bit for bit.
* Poisson sample means hold to the law of large numbers: the mean of y - C e^{-p} over all
  elements is within 5 standard errors of 0, and the open beam's mean is C.
* The noiseless data are exactly rank M (Eq. 3 with w = 0): the (M+1)-th singular value of
  p_true is at fp64 rounding level.
"""
import numpy as np
import torch

import synthdata as sd


def test_eq2_inverts_eq10_without_noise():
    cfg = sd.CONFIGS[1]
    pr = sd.make_problem(cfg, noise=False)
    M = cfg.M
    ptrue = pr["P"].reshape(M, cfg.Np).T.contiguous() @ torch.as_tensor(pr["mu"], dtype=torch.float64)
    y0 = torch.full_like(ptrue, cfg.counts)
    y = sd.expected_counts(ptrue, cfg.counts)
    Y = sd.neglog(y0, y)
    assert float((Y - ptrue).abs().max()) <= 1e-12
    # and the noiseless problem's Y is fp32(p_true)
    assert torch.equal(pr["Y"], ptrue.float())


def test_log_table_and_integer_count_path():
    L = sd.log_table()
    n = np.arange(256)
    assert L[0] == np.log(0.5) and np.allclose(L[1:], np.log(n[1:]), rtol=0, atol=0)
    cfg = sd.CONFIGS[1]
    pr = sd.make_problem(cfg, return_counts=True)
    y0, y = pr["y0"].long(), pr["y"].long()
    Lt = torch.as_tensor(L)
    rc = torch.arange(cfg.Np) % (cfg.Nr * cfg.Nc)
    Yc = (Lt[y0[rc]] - Lt[y]).float()
    assert torch.equal(Yc, pr["Y"])
    # the table path equals Eq. 2 on the integer counts (same fp64 function, up to libm)
    assert float((sd.neglog(y0[rc].double(), y.double()) - (Lt[y0[rc]] - Lt[y])).abs().max()) <= 1e-14


def test_poisson_means_law_of_large_numbers():
    cfg = sd.CONFIGS[1]
    pr = sd.make_problem(cfg, return_counts=True)
    ptrue = pr["P"].reshape(cfg.M, cfg.Np).T.contiguous() @ torch.as_tensor(pr["mu"], dtype=torch.float64)
    lam = sd.expected_counts(ptrue, cfg.counts)
    d = pr["y"].double() - lam
    se = float(torch.sqrt(lam.mean() / d.numel()))
    assert abs(float(d.mean())) <= 5 * se
    ob = pr["y0"].double()
    assert abs(float(ob.mean()) - cfg.counts) <= 5 * np.sqrt(cfg.counts / ob.numel())
    # the minimum mean transmission is about 22% (max line integral 1.5)
    assert abs(float(ptrue.max()) - 1.5) <= 1e-9


def test_noiseless_data_exactly_rank_m():
    cfg = sd.CONFIGS[1]
    pr = sd.make_problem(cfg, noise=False)
    ptrue = pr["P"].reshape(cfg.M, cfg.Np).T.contiguous() @ torch.as_tensor(pr["mu"], dtype=torch.float64)
    s = torch.linalg.svdvals(ptrue)
    assert float(s[cfg.M] / s[0]) <= 1e-13
