"""GPU parity of the counts-domain input (NEXT-1: Eq. 2, Appendix-A offset
PAPER.md:718-725, the 1/2-count floor of DESIGN.md R7) through the C ABI.

* hsnct_counts_to_projections is bit-identical to fp32 of the fp64 oracle
  (oracle.counts_to_projections), with and without the offset b, on the vector (N_k % 4 == 0)
  and scalar paths, into a padded Y.
* The generator's uint8 path: synthdata's Y equals the decoded counts bit for bit.
* hsnct_subspace_decompose_counts equals hsnct_subspace_decompose on the materialised Y bit for
  bit (V, D, objective trace, clamped count) on every row-pass plan: persistent fused (K = 3, 9),
  per-iteration fused, two-pass and tcgen05.
* Errors: non-finite b is a deferred E_DATA; wrong dtypes / shapes are E_ARG.
"""
import numpy as np
import pytest
import torch

import oracle
import synthdata as sd

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")


def counts(cfg, seed):
    g = torch.Generator().manual_seed(seed)
    y0 = torch.poisson(torch.full((cfg.Nr * cfg.Nc, cfg.Nk), cfg.counts, dtype=torch.float64), generator=g)
    y = torch.poisson(torch.full((cfg.Np, cfg.Nk), 0.5 * cfg.counts, dtype=torch.float64), generator=g)
    return y.clamp(max=255).to(torch.uint8), y0.clamp(max=255).to(torch.uint8)


@pytest.mark.parametrize("Nk,with_b", [(40, False), (40, True), (203, True), (1600, False)])
def test_counts_to_projections_bitwise(Nk, with_b):
    from paper_2410_22500_b200 import Hsnct
    cfg = sd.custom(idx=40 + Nk, Nc=12, Nv=5, Nr=3, Nk=Nk, K=2, M=2, counts=20.0)
    y, y0 = counts(cfg, Nk)
    b = torch.randn((cfg.Nv, cfg.Nk), generator=torch.Generator().manual_seed(1)).float() if with_b else None
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    ld = Nk + 5
    Ybuf = torch.full((cfg.Np, ld), 7.0, dtype=torch.float32, device=DEV)
    Y = h.counts_to_projections(y.to(DEV), y0.to(DEV), None if b is None else b.to(DEV), Y=Ybuf[:, :Nk])
    h.sync()
    P = oracle.counts_to_projections(y.numpy(), y0.numpy(), cfg.Nv, None if b is None else b.double().numpy())
    assert np.array_equal(Y.cpu().numpy(), P.astype(np.float32))
    assert torch.all(Ybuf[:, Nk:] == 7.0)   # padding untouched
    h.close()


def test_generator_counts_decode_bitwise():
    from paper_2410_22500_b200 import Hsnct
    cfg = sd.custom(idx=51, Nc=24, Nv=10, Nr=2, Nk=200, K=3, M=3, counts=20.0)
    pr = sd.make_problem(cfg, return_counts=True)
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    Y = h.counts_to_projections(pr["y"].to(DEV), pr["y0"].to(DEV))
    h.sync()
    assert torch.equal(Y.cpu(), pr["Y"])
    h.close()


@pytest.mark.parametrize("plan,cfg", [
    (None, sd.custom(idx=52, Nc=24, Nv=10, Nr=2, Nk=200, K=3, M=3, counts=20.0)),
    (None, sd.custom(idx=53, Nc=32, Nv=16, Nr=2, Nk=1200, K=9, M=3, counts=20.0)),
    ("nopersist", sd.custom(idx=54, Nc=20, Nv=13, Nk=203, K=5, M=4, counts=30.0)),
    ("twopass", sd.custom(idx=55, Nc=20, Nv=13, Nk=203, K=5, M=4, counts=30.0)),
    ("tc", sd.CONFIGS[1]),
    ("mma", sd.custom(idx=56, Nc=20, Nv=13, Nk=203, K=5, M=4, counts=30.0)),
    ("mma", sd.custom(idx=57, Nc=24, Nv=10, Nr=3, Nk=400, K=6, M=4, counts=20.0)),  # vector decode (N_k % 8 == 0)
])
def test_decompose_counts_bitwise(monkeypatch, plan, cfg):
    if plan == "nopersist":
        monkeypatch.setenv("HSNCT_NO_PERSIST", "1")
    elif plan is not None:
        monkeypatch.setenv("HSNCT_NMF", plan)
    from paper_2410_22500_b200 import Hsnct
    pr = sd.make_problem(cfg, return_counts=True)
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    n = 12
    b = (0.05 * torch.randn((cfg.Nv, cfg.Nk), generator=torch.Generator().manual_seed(2))).float().to(DEV)
    y, y0 = pr["y"].to(DEV), pr["y0"].to(DEV)
    outs = []
    for mode in ("materialised", "counts"):
        V, D = pr["V0"].to(DEV).clone(), pr["D0"].to(DEV).clone()
        obj = torch.zeros(2 * n, dtype=torch.float64, device=DEV)
        if mode == "materialised":
            Ybuf = torch.empty((cfg.Np, (cfg.Nk + 3) // 4 * 4), dtype=torch.float32, device=DEV)
            Y = h.counts_to_projections(y, y0, b, Y=Ybuf[:, :cfg.Nk])
            h.subspace_decompose(Y, V, D, n, obj_trace=obj)
        else:
            h.subspace_decompose_counts(y, y0, V, D, n, b=b, obj_trace=obj)
        h.sync()
        outs.append((V, D, obj, h.decompose_stats()["n_clamped"]))
    (V1, D1, o1, c1), (V2, D2, o2, c2) = outs
    print(h.debug_plan())
    assert torch.equal(V1, V2) and torch.equal(D1, D2) and torch.equal(o1, o2) and c1 == c2
    assert c1 > 0
    # and the materialised path itself is the oracle's NMF on the decoded Y (as everywhere else)
    Yo = oracle.counts_to_projections(pr["y"].numpy(), pr["y0"].numpy(), cfg.Nv, b.double().cpu().numpy())
    Vo, Do = oracle.nmf(Yo.astype(np.float32), pr["V0"].numpy(), pr["D0"].numpy(), n)
    assert float(torch.linalg.norm(V2.cpu().double() - torch.from_numpy(Vo)) / np.linalg.norm(Vo)) <= 1e-3
    h.close()


def test_counts_errors():
    from paper_2410_22500_b200 import Hsnct, HsnctError
    cfg = sd.custom(idx=56, Nc=12, Nv=5, Nr=2, Nk=40, K=2, M=2, counts=20.0)
    y, y0 = counts(cfg, 3)
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    b = torch.zeros((cfg.Nv, cfg.Nk), dtype=torch.float32, device=DEV)
    b[2, 7] = float("nan")
    h.counts_to_projections(y.to(DEV), y0.to(DEV), b)
    with pytest.raises(HsnctError) as ei:
        h.sync()
    assert ei.value.status == 2
    with pytest.raises(HsnctError):
        h.counts_to_projections(y.to(DEV).float(), y0.to(DEV))
    with pytest.raises(HsnctError):
        h.counts_to_projections(y.to(DEV), y0.to(DEV)[:-1])
    h.close()


@pytest.mark.parametrize("plan", [None, "mma", "twopass"])
def test_fhr_stream_counts_equals_fhr_stream(monkeypatch, plan):
    """hsnct_fhr_stream_counts (NEXT-1 end to end): host uint8 counts and the offset b in, Eq. 2
    on the device; every x^h window and V, D equal hsnct_fhr_stream on the decoded Y bit for bit
    (plans that decode in their preparation, and the two-pass plan that decodes into a Y buffer)."""
    if plan is not None:
        monkeypatch.setenv("HSNCT_NMF", plan)
    from paper_2410_22500_b200 import Hsnct
    cfg = sd.custom(idx=58, Nc=24, Nv=10, Nr=3, Nk=96, K=4, M=3, counts=20.0)
    pr = sd.make_problem(cfg, return_counts=True)
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    b = (0.05 * torch.randn((cfg.Nv, cfg.Nk), generator=torch.Generator().manual_seed(4))).float()
    Ybuf = torch.empty((cfg.Np, (cfg.Nk + 3) // 4 * 4), dtype=torch.float32, device=DEV)
    Y = h.counts_to_projections(pr["y"].to(DEV), pr["y0"].to(DEV), b.to(DEV), Y=Ybuf[:, :cfg.Nk]).cpu()
    out = {}
    for mode in ("Y", "counts"):
        wins = []
        Vh, Dh = torch.empty_like(pr["V0"]), torch.empty_like(pr["D0"])

        def on_window(s0, ns, xh):
            wins.append((s0, ns, xh.clone()))
        if mode == "Y":
            h.fhr_stream(Y.pin_memory(), pr["V0"], pr["D0"], 12, window_slices=2, on_window=on_window, V=Vh, D=Dh)
        else:
            h.fhr_stream_counts(pr["y"].pin_memory(), pr["y0"].pin_memory(), pr["V0"], pr["D0"], 12, b=b.pin_memory(),
                                window_slices=2, on_window=on_window, V=Vh, D=Dh)
        out[mode] = (wins, Vh, Dh)
    (w1, V1, D1), (w2, V2, D2) = out["Y"], out["counts"]
    print(h.debug_plan())
    assert torch.equal(V1, V2) and torch.equal(D1, D2)
    assert [(s, n) for s, n, _ in w1] == [(s, n) for s, n, _ in w2] == [(0, 2), (2, 1)]
    for (_, _, x1), (_, _, x2) in zip(w1, w2):
        assert torch.equal(x1, x2)
    h.close()
