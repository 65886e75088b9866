"""GPU parity of the mma.sync row pass (nmf_mma.cu) against the fp64 oracle.

HSNCT_NMF=mma forces the plan at handle creation, so these shapes -- small enough for the
oracle -- run the kernel templates the bench runs: every K in 1..8, N_k giving 1..13 16-bin
blocks per warp (every NBW instance, warps without blocks when N_k < 128), ragged N_k (not a
multiple of 16) and ragged N_p (a partial last 16-row tile), the first-iteration V0 check and
the non-finite / all-zero data errors, bitwise determinism, and a resumed decomposition.

Tolerance: 1e-3 relative L2 on V and D (BASELINE.json north_star), objective rtol 1e-3.  The
fp16 hi/lo split keeps products fp32-accurate (2^-22); the measured drift is ~1e-6.
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
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture
def mm(monkeypatch):
    monkeypatch.setenv("HSNCT_NMF", "mma")
    from paper_2410_22500_b200 import Hsnct

    def make(cfg):
        h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
        assert h.debug_plan().startswith("mma "), h.debug_plan()
        return h
    return make


def padded(Y, ld):
    buf = torch.full((Y.shape[0], ld), float("nan"), dtype=torch.float32, device=DEV)
    buf[:, :Y.shape[1]] = Y.to(DEV)
    return buf[:, :Y.shape[1]]


CASES = [
    (sd.CONFIGS[1], 100),                                         # Nk=200: one chunk per rank
    (sd.custom(idx=51, Nc=20, Nv=13, Nk=203, K=5, M=4), 40),      # ragged Nk and Np (260 rows)
    (sd.custom(idx=52, Nc=17, Nv=9, Nk=64, K=1, M=2), 30),        # K=1, 16 bins per rank
    (sd.custom(idx=53, Nc=24, Nv=10, Nr=3, Nk=501, K=2, M=2), 25),
    (sd.custom(idx=54, Nc=32, Nv=16, Nr=2, Nk=1600, K=6, M=6), 20),   # the C3-C5 range split (7 chunks)
    (sd.custom(idx=55, Nc=32, Nv=12, Nr=2, Nk=1200, K=4, M=4), 20),   # the C2 split (5 chunks)
    (sd.custom(idx=56, Nc=24, Nv=11, Nr=1, Nk=1650, K=8, M=4), 10),   # 13 blocks per warp, ragged, K=8
    (sd.custom(idx=57, Nc=40, Nv=9, Nr=1, Nk=333, K=7, M=5), 15),
    (sd.custom(idx=58, Nc=16, Nv=8, Nr=1, Nk=96, K=3, M=3), 12),
    (sd.custom(idx=59, Nc=13, Nv=7, Nr=1, Nk=40, K=2, M=2), 12),     # 3 blocks: warps without bins
    (sd.custom(idx=70, Nc=24, Nv=9, Nr=2, Nk=1664, K=6, M=5), 10),    # 13 blocks on every warp
    # K = 9..16: two column blocks of 8 components (the paper's N_s = 9, Table I)
    (sd.custom(idx=75, Nc=32, Nv=16, Nr=2, Nk=1200, K=9, M=3), 15),   # the C6 shape class
    (sd.custom(idx=76, Nc=20, Nv=13, Nk=203, K=12, M=5), 12),         # ragged N_k and N_p
    (sd.custom(idx=77, Nc=24, Nv=10, Nr=2, Nk=1280, K=16, M=6), 8),   # K = 16 (per-iteration launches)
    (sd.custom(idx=78, Nc=16, Nv=9, Nr=1, Nk=64, K=10, M=4), 10),     # 4 blocks: warps without bins
]


@pytest.mark.parametrize("cfg,n_iter", CASES)
def test_mma_nmf_parity(mm, cfg, n_iter):
    pr = sd.make_problem(cfg)
    h = mm(cfg)
    Yd = padded(pr["Y"], ((cfg.Nk + 3) // 4) * 4 + 4)
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    obj = torch.zeros(2 * n_iter, dtype=torch.float64, device=DEV)
    h.subspace_decompose(Yd, V, D, n_iter, obj_trace=obj)
    h.sync()
    Vo, Do, objo = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), n_iter, objective=True)
    eV, eD = rel(V, Vo), rel(D, Do)
    print(f"{cfg.describe()} {n_iter} it: V {eV:.2e} D {eD:.2e}")
    assert eV <= 1e-3 and eD <= 1e-3, (eV, eD)
    ob = obj.cpu().numpy()
    np.testing.assert_allclose(ob, objo, rtol=1e-3)
    assert np.all(np.diff(ob) <= 1e-5 * np.abs(ob[:-1]))


def test_mma_one_step_tight(mm):
    """One iteration from the init at N_k = 1600 (13 blocks per warp): the hi/lo products are fp32-accurate,
    so V_1 and D_1 agree with the oracle to ~1e-6, far inside the 1e-3 budget."""
    cfg = sd.custom(idx=60, Nc=64, Nv=16, Nr=2, Nk=1600, K=6, M=6)
    pr = sd.make_problem(cfg)
    h = mm(cfg)
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    h.subspace_decompose(pr["Y"].to(DEV), V, D, 1)
    h.sync()
    Vo, Do = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), 1)
    assert rel(V, Vo) <= 2e-5 and rel(D, Do) <= 2e-5, (rel(V, Vo), rel(D, Do))


def test_mma_deterministic_and_resumable(mm):
    cfg = sd.custom(idx=61, Nc=32, Nv=16, Nr=3, Nk=800, K=6, M=5)
    pr = sd.make_problem(cfg)
    h = mm(cfg)
    Y = pr["Y"].to(DEV)
    outs = []
    for split in ((20,), (20,), (20,), (7, 13)):
        V = pr["V0"].to(DEV).clone()
        D = pr["D0"].to(DEV).clone()
        for n in split:
            h.subspace_decompose(Y, V, D, n)
        h.sync()
        outs.append((V.cpu(), D.cpu()))
    for V, D in outs[1:]:  # one launch per iteration and a fixed schedule: resume is bitwise too
        assert torch.equal(V, outs[0][0]) and torch.equal(D, outs[0][1])


def test_mma_data_errors(mm):
    from paper_2410_22500_b200 import HsnctError
    cfg = sd.custom(idx=62, Nc=16, Nv=8, Nk=96, K=2)
    h = mm(cfg)
    Y = torch.rand((cfg.Np, cfg.Nk), device=DEV)
    V = torch.rand((cfg.Np, 2), device=DEV) + 0.1
    D = torch.rand((2, cfg.Nk), device=DEV) + 0.1
    Yn = Y.clone()
    Yn[3, 4] = float("nan")
    h.subspace_decompose(Yn, V.clone(), D.clone(), 2)
    with pytest.raises(HsnctError) as e:
        h.sync()
    assert e.value.status == 2 and "non-finite" in str(e.value)
    h.subspace_decompose(-Y, V.clone(), D.clone(), 2)
    with pytest.raises(HsnctError) as e:
        h.sync()
    assert e.value.status == 2 and "identically zero" in str(e.value)
    Vn = V.clone()
    Vn[5, 1] = -1.0
    h.subspace_decompose(Y, Vn, D.clone(), 1)
    with pytest.raises(HsnctError) as e:
        h.sync()
    assert e.value.status == 2 and "V0/D0" in str(e.value)
    h.subspace_decompose(Y, V.clone(), D.clone(), 3)
    h.sync()


def test_mma_scale_invariance(mm):
    """Scaling Y by 2^20 or 2^-20 scales V D by the same factor exactly in exact arithmetic;
    the power-of-two operand scales keep the fp16 split in range either way."""
    cfg = sd.custom(idx=63, Nc=16, Nv=8, Nr=2, Nk=160, K=3, M=3)
    pr = sd.make_problem(cfg)
    h = mm(cfg)
    res = []
    for s in (1.0, 2.0 ** 20, 2.0 ** -20):
        V = (pr["V0"] * np.sqrt(s)).to(DEV)
        D = (pr["D0"] * np.sqrt(s)).to(DEV)
        h.subspace_decompose((pr["Y"] * s).to(DEV), V, D, 10)
        h.sync()
        res.append((V.cpu() / np.sqrt(s), D.cpu() / np.sqrt(s)))
    for V, D in res[1:]:
        assert rel(V, res[0][0].numpy()) <= 1e-5 and rel(D, res[0][1].numpy()) <= 1e-5


@pytest.mark.parametrize("plan", ["mma", "ffma"])
def test_nmf_stage_timing(monkeypatch, plan):
    """hsnct_debug_nmf_timing/_times: events around the input preparation and the iterations
    (the persistent launch), same result as an untimed call."""
    monkeypatch.setenv("HSNCT_NMF", plan)
    from paper_2410_22500_b200 import Hsnct, HsnctError
    cfg = sd.custom(idx=79, Nc=32, Nv=16, Nr=2, Nk=400, K=5, M=4)
    pr = sd.make_problem(cfg)
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    Y = pr["Y"].to(DEV)
    out = []
    for timed in (False, True):
        V, D = pr["V0"].to(DEV).clone(), pr["D0"].to(DEV).clone()
        h.debug_nmf_timing(timed)
        h.subspace_decompose(Y, V, D, 6)
        if timed:
            prep_ms, it_ms = h.debug_nmf_times()
            assert prep_ms > 0 and it_ms > 0
        h.sync()
        out.append((V.cpu(), D.cpu()))
    h.debug_nmf_timing(False)
    assert torch.equal(out[0][0], out[1][0]) and torch.equal(out[0][1], out[1][1])
    with pytest.raises(HsnctError):
        h.debug_nmf_times()


def test_mma_per_iteration_launches_match_persistent(monkeypatch):
    """HSNCT_NO_PERSIST=1: the same pass as one launch per iteration + k_dred (the path taken
    when the cooperative launch is refused, by the sharded row pass, and for K*K + K*SL > 256);
    against the oracle and against the persistent launch (same row-pass arithmetic, different
    reduction order in the D update)."""
    cfg = sd.custom(idx=80, Nc=32, Nv=16, Nr=2, Nk=800, K=6, M=5)
    pr = sd.make_problem(cfg)
    monkeypatch.setenv("HSNCT_NMF", "mma")
    from paper_2410_22500_b200 import Hsnct
    res = []
    for nop in ("0", "1"):
        monkeypatch.setenv("HSNCT_NO_PERSIST", nop)
        h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
        assert ("PERSIST=1" in h.debug_plan()) == (nop == "0"), h.debug_plan()
        V, D = pr["V0"].to(DEV).clone(), pr["D0"].to(DEV).clone()
        obj = torch.zeros(40, dtype=torch.float64, device=DEV)
        h.subspace_decompose(pr["Y"].to(DEV), V, D, 20, obj_trace=obj)
        h.sync()
        res.append((V, D, obj))
        h.close()
    Vo, Do, objo = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), 20, objective=True)
    for V, D, obj in res:
        assert rel(V, Vo) <= 1e-3 and rel(D, Do) <= 1e-3
        np.testing.assert_allclose(obj.cpu().numpy(), objo, rtol=1e-3)
    assert rel(res[0][0], res[1][0].cpu().double().numpy()) <= 1e-5


@pytest.mark.parametrize("Nc,Nv,Nr,Nk,K", [(3, 2, 1, 5, 2), (4, 3, 1, 17, 1), (5, 3, 1, 33, 9)])
def test_mma_degenerate_shapes(mm, Nc, Nv, Nr, Nk, K):
    """Fewer rows than one 16-row tile (one ragged tile, one CTA), N_k below one 16-bin block per
    warp, K = 1 and two column blocks with a single extra component."""
    cfg = sd.custom(idx=90 + Nc, Nc=Nc, Nv=Nv, Nr=Nr, Nk=Nk, K=K, M=min(K, 2))
    pr = sd.make_problem(cfg)
    h = mm(cfg)
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    h.subspace_decompose(padded(pr["Y"], (Nk + 3) // 4 * 4), V, D, 8)
    h.sync()
    Vo, Do = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), 8)
    assert rel(V, Vo) <= 1e-4 and rel(D, Do) <= 1e-4, (rel(V, Vo), rel(D, Do))


@pytest.mark.parametrize("cfg,n_iter", [c for c in CASES if c[0].K > 8] +
                         [(sd.custom(idx=79, Nc=5, Nv=3, Nr=1, Nk=33, K=9, M=2), 8)])
def test_mma_sixteen_warps(monkeypatch, mm, cfg, n_iter):
    """K = 9..16 on the experimental 16-warp form (a -DHSNCT_MMA_MW16 build with HSNCT_MMA_MW=16: <= 5 blocks per warp, the half-warps
    of the V update summing warps 0-7 and 8-15's partials): same parity bar, and the result agrees
    with the default 8-warp form to fp32 summation order."""
    pr = sd.make_problem(cfg)
    out = []
    for mw in ("16", "8"):
        monkeypatch.setenv("HSNCT_MMA_MW", mw)
        h = mm(cfg)
        if mw == "16" and "MW=16" not in h.debug_plan():
            pytest.skip("the 16-warp form is not in this build (build.py --variant=mw16 -DHSNCT_MMA_MW16)")
        assert ("MW=16" in h.debug_plan()) == (mw == "16"), h.debug_plan()
        V = pr["V0"].to(DEV).clone()
        D = pr["D0"].to(DEV).clone()
        h.subspace_decompose(padded(pr["Y"], ((cfg.Nk + 3) // 4) * 4 + 4), V, D, n_iter)
        h.sync()
        h.close()
        out.append((V, D))
    Vo, Do = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), n_iter)
    for V, D in out:
        assert rel(V, Vo) <= 1e-3 and rel(D, Do) <= 1e-3, (rel(V, Vo), rel(D, Do))
    assert rel(out[0][0], out[1][0].cpu().double().numpy()) <= 1e-4
