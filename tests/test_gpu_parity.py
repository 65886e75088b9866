"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle on the same
seeded inputs.  Tolerances (BASELINE.json north_star):
  FBP and synthesis  <= 1e-4 relative L2;
  NMF (fixed init, fixed iteration count) <= 1e-3 relative L2 on V, D and x^h.
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
    b = b.detach().cpu().double().numpy() if isinstance(b, torch.Tensor) else np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def H():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2410_22500_b200 import Hsnct, lib
    lib()

    def make(cfg, angles=None):
        return Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, angles=angles, device=0)
    return make


def padded(Y, ld, fill=float("nan")):
    """Y on the device with ld >= Nk, padding columns poisoned (must be ignored)."""
    Np, Nk = Y.shape
    buf = torch.full((Np, ld), fill, dtype=torch.float32, device=DEV)
    buf[:, :Nk] = Y.to(DEV)
    return buf[:, :Nk]


# ---------------------------------------------------------------------- NMF
@pytest.mark.parametrize("cfg,n_iter", [
    (sd.CONFIGS[1], 100),
    (sd.custom(idx=7, Nc=20, Nv=13, Nk=203, K=5, M=4), 40),     # ragged N_p, N_k % 4 != 0
    (sd.custom(idx=8, Nc=17, Nv=9, Nk=37, K=1, M=2), 30),       # K = 1
    (sd.custom(idx=9, Nc=24, Nv=10, Nr=3, Nk=64, K=16, M=5), 25),  # K = 16, several slices
    # three groups with a row-split last lambda slot (17 pairs past 3 x 128), ragged N_k
    (sd.custom(idx=23, Nc=24, Nv=11, Nr=1, Nk=801, K=6, M=6), 20),
    # K*K = 64 > 32: the objective reads G_old across several warps
    (sd.custom(idx=24, Nc=24, Nv=11, Nr=1, Nk=200, K=8, M=4), 10),
    # K = 9 .. 12 on the fused persistent kernel (the paper's N_s = 9, Table I shape's N_k)
    (sd.custom(idx=25, Nc=32, Nv=16, Nr=4, Nk=1200, K=9, M=3), 20),
    (sd.custom(idx=26, Nc=24, Nv=11, Nr=2, Nk=600, K=12, M=5), 12),
    (sd.custom(idx=27, Nc=20, Nv=9, Nr=1, Nk=333, K=10, M=4), 12),
    # few rows, long spectra: the persistent kernel's D-update slice would not fit,
    # the plan takes the per-iteration launches
    (sd.custom(idx=28, Nc=16, Nv=8, Nr=1, Nk=1600, K=6, M=3), 10),
    (sd.custom(idx=29, Nc=8, Nv=2, Nr=1, Nk=2048, K=3, M=2), 10),
    (sd.custom(idx=30, Nc=12, Nv=4, Nr=1, Nk=1200, K=12, M=2), 8),
])
def test_nmf_parity(H, cfg, n_iter):
    pr = sd.make_problem(cfg)
    h = H(cfg)
    Yd = padded(pr["Y"], ((cfg.Nk + 3) // 4) * 4 + 4)
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    obj = torch.zeros(2 * n_iter, dtype=torch.float64, device=DEV)
    h.subspace_decompose(Yd, V, D, n_iter, obj_trace=obj)
    h.sync()
    Vo, Do, objo = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), n_iter, objective=True)
    assert rel(V, Vo) <= 1e-3, rel(V, Vo)
    assert rel(D, Do) <= 1e-3, rel(D, Do)
    ob = obj.cpu().numpy()
    np.testing.assert_allclose(ob, objo, rtol=1e-3)
    assert np.all(np.diff(ob) <= 1e-5 * np.abs(ob[:-1]))


def test_nmf_parity_c2_shape(H):
    cfg = sd.CONFIGS[2]
    pr = sd.make_problem(cfg)
    h = H(cfg)
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    n = 12
    h.subspace_decompose(pr["Y"].to(DEV), V, D, n)
    h.sync()
    Vo, Do = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), n)
    assert rel(V, Vo) <= 1e-3 and rel(D, Do) <= 1e-3, (rel(V, Vo), rel(D, Do))


def test_nmf_deterministic_and_resumable(H):
    cfg = sd.CONFIGS[1]
    pr = sd.make_problem(cfg)
    h = H(cfg)
    Y = pr["Y"].to(DEV)
    outs = []
    # the tile order alternates per iteration within a call, so a
    # resume after an even number of iterations is bitwise; after an odd number it
    # differs only by fp32 summation order
    for split in ((30,), (30,), (12, 18), (11, 19)):
        V = pr["V0"].to(DEV).clone()
        D = pr["D0"].to(DEV).clone()
        for n in split:
            h.subspace_decompose(Y, V, D, n)
        h.sync()
        outs.append((V.cpu(), D.cpu()))
    for V, D in outs[1:3]:
        assert torch.equal(V, outs[0][0]) and torch.equal(D, outs[0][1])
    assert rel(outs[3][0], outs[0][0]) < 1e-5 and rel(outs[3][1], outs[0][1]) < 1e-5


@pytest.mark.parametrize("cfg,n_iter", [(sd.custom(idx=14, Nc=32, Nv=16, Nr=4, Nk=1200, K=9, M=3), 12),
                                        (sd.custom(idx=15, Nc=24, Nv=11, Nr=2, Nk=203, K=16, M=5), 10),
                                        (sd.custom(idx=16, Nc=20, Nv=13, Nk=203, K=5, M=4), 10)])
def test_nmf_twopass_plan(monkeypatch, cfg, n_iter):
    """HSNCT_NMF=twopass: the k_vstep + k_bpart + k_dred kernels (the fallback for shapes the
    fused kernel cannot hold) against the oracle, K = 5, 9, 16."""
    monkeypatch.setenv("HSNCT_NMF", "twopass")
    from paper_2410_22500_b200 import Hsnct
    pr = sd.make_problem(cfg)
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    assert h.debug_plan().startswith("twopass"), h.debug_plan()
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    obj = torch.zeros(2 * n_iter, dtype=torch.float64, device=DEV)
    h.subspace_decompose(padded(pr["Y"], ((cfg.Nk + 3) // 4) * 4), V, D, n_iter, obj_trace=obj)
    h.sync()
    Vo, Do, objo = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), n_iter, objective=True)
    assert rel(V, Vo) <= 1e-3 and rel(D, Do) <= 1e-3, (rel(V, Vo), rel(D, Do))
    np.testing.assert_allclose(obj.cpu().numpy(), objo, rtol=1e-3)
    h.close()


@pytest.mark.parametrize("cfg,n_iter", [(sd.CONFIGS[1], 60),
                                        (sd.custom(idx=11, Nc=20, Nv=13, Nk=203, K=5, M=4), 25),
                                        (sd.custom(idx=12, Nc=32, Nv=16, Nr=4, Nk=1200, K=9, M=3), 15),
                                        (sd.custom(idx=13, Nc=24, Nv=11, Nr=2, Nk=600, K=12, M=5), 10)])
def test_nmf_per_iteration_fallback(H, monkeypatch, cfg, n_iter):
    """The per-iteration launch path (used when a cooperative launch is refused)."""
    monkeypatch.setenv("HSNCT_NO_PERSIST", "1")
    pr = sd.make_problem(cfg)
    h = H(cfg)
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    obj = torch.zeros(2 * n_iter, dtype=torch.float64, device=DEV)
    l0 = h.kernel_launches
    h.subspace_decompose(padded(pr["Y"], ((cfg.Nk + 3) // 4) * 4), V, D, n_iter, obj_trace=obj)
    h.sync()
    assert h.kernel_launches - l0 >= 2 * n_iter  # really the per-iteration path
    Vo, Do, objo = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), n_iter, objective=True)
    assert rel(V, Vo) <= 1e-3 and rel(D, Do) <= 1e-3, (rel(V, Vo), rel(D, Do))
    np.testing.assert_allclose(obj.cpu().numpy(), objo, rtol=1e-3)


def test_nmf_fixed_point(H):
    cfg = sd.custom(idx=10, Nc=16, Nv=8, Nk=24, K=3)
    h = H(cfg)
    g = torch.Generator().manual_seed(3)
    Vs = torch.randint(1, 5, (cfg.Np, 3), generator=g).float()
    Ds = torch.randint(1, 5, (3, cfg.Nk), generator=g).float()
    Y = (Vs @ Ds).to(DEV)
    V, D = Vs.to(DEV).clone(), Ds.to(DEV).clone()
    h.subspace_decompose(Y, V, D, 10)
    h.sync()
    assert rel(V, Vs) < 1e-6 and rel(D, Ds) < 1e-6


def test_nmf_zero_iterations_noop(H):
    cfg = sd.CONFIGS[1]
    pr = sd.make_problem(cfg)
    h = H(cfg)
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    h.subspace_decompose(pr["Y"].to(DEV), V, D, 0)
    h.sync()
    assert torch.equal(V.cpu(), pr["V0"]) and torch.equal(D.cpu(), pr["D0"])


# ---------------------------------------------------------------------- FBP
@pytest.mark.parametrize("cfg", [
    sd.CONFIGS[1],
    sd.custom(idx=11, Nc=63, Nv=37, Nr=2, Nk=10, K=5),
    sd.custom(idx=12, Nc=100, Nv=45, Nr=1, Nk=20, K=16),
    sd.custom(idx=13, Nc=33, Nv=8, Nr=3, Nk=4, K=1),
    sd.custom(idx=26, Nc=300, Nv=9, Nr=2, Nk=6, K=5),   # P = 1024 (32 x 32 four-step FFT), KC = 5
    sd.custom(idx=27, Nc=130, Nv=12, Nr=1, Nk=8, K=7),  # P = 512, KC = 7 (scalar window loads)
])
def test_fbp_parity(H, cfg):
    g = torch.Generator().manual_seed(cfg.idx)
    V = torch.rand((cfg.Np, cfg.K), generator=g)
    h = H(cfg)
    X = h.fbp(V.to(DEV))
    torch.cuda.synchronize()
    Xo = oracle.fbp(V.numpy(), cfg.Nv, cfg.Nr, cfg.Nc)
    assert rel(X, Xo) <= 1e-4, rel(X, Xo)


def test_fbp_and_dhr_large_detector(H):
    """N_c = 600 -> P = 2048: the shared-memory radix-2 ramp filter (P > 1024) and, for DHR,
    8-bin channel chunks (backprojection KC = 8)."""
    cfg = sd.custom(idx=25, Nc=600, Nv=7, Nr=1, Nk=11, K=3)
    g = torch.Generator().manual_seed(8)
    V = torch.rand((cfg.Np, cfg.K), generator=g)
    h = H(cfg)
    X = h.fbp(V.to(DEV))
    Y = torch.rand((cfg.Np, cfg.Nk), generator=g) - 0.1
    Xh = h.dhr(padded(Y, 12), 0, 1, 1, 9)
    torch.cuda.synchronize()
    Xo = oracle.fbp(V.numpy(), cfg.Nv, cfg.Nr, cfg.Nc)
    assert rel(X, Xo) <= 1e-4, rel(X, Xo)
    Xho = oracle.dhr(Y.numpy(), cfg.Nv, cfg.Nr, cfg.Nc, slice0=0, n_slices=1, bin0=1, n_bins=9)
    assert rel(Xh, Xho) <= 1e-4, rel(Xh, Xho)


def test_fbp_stage_timing(H):
    """hsnct_debug_fbp_timing/_times: events around the two launches, same result."""
    from paper_2410_22500_b200.hsnct import HsnctError
    cfg = sd.custom(idx=22, Nc=64, Nv=30, Nr=2, Nk=8, K=6)
    V = torch.rand((cfg.Np, cfg.K), generator=torch.Generator().manual_seed(3)).to(DEV)
    h = H(cfg)
    X0 = h.fbp(V)
    h.debug_fbp_timing(True)
    X1 = h.fbp(V)
    ramp_ms, bp_ms = h.debug_fbp_times()
    h.debug_fbp_timing(False)
    assert ramp_ms > 0 and bp_ms > 0
    assert torch.equal(X0, X1)
    with pytest.raises(HsnctError):
        h.debug_fbp_times()


def test_fbp_custom_angles(H):
    cfg = sd.custom(idx=14, Nc=40, Nv=17, Nk=6, K=3)
    ang = np.sort(np.random.default_rng(2).uniform(0, math.pi, cfg.Nv))
    V = torch.rand((cfg.Np, cfg.K), generator=torch.Generator().manual_seed(1))
    h = H(cfg, angles=ang)
    X = h.fbp(V.to(DEV))
    torch.cuda.synchronize()
    Xo = oracle.fbp(V.numpy(), cfg.Nv, cfg.Nr, cfg.Nc, angles=ang)
    assert rel(X, Xo) <= 1e-4


def test_fbp_single_view_impulse_pin(H):
    """Closed form: one impulse at theta = 0 gives (pi/Nv) h[j - c0] in every row."""
    cfg = sd.custom(idx=15, Nc=32, Nv=6, Nk=1, K=1)
    V = torch.zeros((cfg.Np, 1))
    c0 = 9
    V[c0, 0] = 1.0  # view 0, row 0, column c0
    h = H(cfg)
    X = h.fbp(V.to(DEV)).cpu()[0, 0].double().numpy()
    hk = np.array([oracle.ramp_kernel(j - c0) for j in range(cfg.Nc)])
    np.testing.assert_allclose(X, np.tile(math.pi / cfg.Nv * hk, (cfg.Nc, 1)), atol=2e-7)


def test_fbp_analytic_disk(H):
    Nc, Nv = 256, 180
    cfg = sd.custom(idx=16, Nc=Nc, Nv=Nv, Nk=1, K=1)
    th = torch.as_tensor(sd.view_angles(Nv), dtype=torch.float64)[:, None]
    t = (torch.arange(Nc, dtype=torch.float64) - 0.5 * (Nc - 1))[None, :]
    P = sd.ellipse_line_integrals(th, t, 0.0, 0.0, 0.3 * Nc, 0.3 * Nc, 0.0)
    h = H(cfg)
    X = h.fbp(P.float().reshape(-1, 1).to(DEV)).cpu()[0, 0].double().numpy()
    yy, xx = np.mgrid[0:Nc, 0:Nc] - 0.5 * (Nc - 1)
    assert X[np.hypot(xx, yy) < 0.24 * Nc].mean() == pytest.approx(1.0, abs=3e-3)


# ---------------------------------------------------------------- synthesis
@pytest.mark.parametrize("window", [(0, None, 0, None), (1, 2, 3, 17), (2, 1, 5, 3)])
def test_synthesize_parity(H, window):
    cfg = sd.custom(idx=17, Nc=12, Nv=5, Nr=4, Nk=41, K=6)
    g = torch.Generator().manual_seed(4)
    X = torch.randn((cfg.K, cfg.Nr, cfg.Nc, cfg.Nc), generator=g)
    D = torch.rand((cfg.K, cfg.Nk), generator=g)
    s0, ns, b0, nb = window
    ns = cfg.Nr - s0 if ns is None else ns
    nb = cfg.Nk - b0 if nb is None else nb
    h = H(cfg)
    Xh = h.synthesize(X.to(DEV), D.to(DEV), s0, ns, b0, nb)
    torch.cuda.synchronize()
    Xo = oracle.synthesize(X.numpy(), D.numpy(), s0, ns, b0, nb)
    assert rel(Xh, Xo) <= 1e-6


def test_synthesize_strided_unaligned_output(H):
    cfg = sd.custom(idx=18, Nc=8, Nv=5, Nr=2, Nk=30, K=4)
    g = torch.Generator().manual_seed(5)
    X = torch.randn((cfg.K, cfg.Nr, cfg.Nc, cfg.Nc), generator=g).to(DEV)
    D = torch.rand((cfg.K, cfg.Nk), generator=g).to(DEV)
    big = torch.full((cfg.Nx, 33), -7.0, device=DEV)
    out = big[:, 1:1 + 29]            # ld = 33, misaligned base
    h = H(cfg)
    h.synthesize(X, D, 0, cfg.Nr, 1, 29, Xh=out)
    torch.cuda.synchronize()
    Xo = oracle.synthesize(X.cpu().numpy(), D.cpu().numpy(), 0, cfg.Nr, 1, 29)
    assert rel(out, Xo) <= 1e-6
    assert torch.all(big[:, 0] == -7.0) and torch.all(big[:, 30:] == -7.0)


def test_synthesize_empty_window(H):
    cfg = sd.custom(idx=19, Nc=8, Nv=5, Nr=2, Nk=30, K=4)
    h = H(cfg)
    X = torch.zeros((cfg.K, cfg.Nr, cfg.Nc, cfg.Nc), device=DEV)
    D = torch.zeros((cfg.K, cfg.Nk), device=DEV)
    out = h.synthesize(X, D, 1, 0, 0, 5)
    assert out.numel() == 0


# ---------------------------------------------------------------------- DHR
@pytest.mark.parametrize("cfg,window", [
    (sd.CONFIGS[1], (0, 1, 0, 40)),
    (sd.custom(idx=20, Nc=50, Nv=21, Nr=3, Nk=37, K=2), (1, 2, 3, 33)),
])
def test_dhr_parity(H, cfg, window):
    pr = sd.make_problem(cfg)
    s0, ns, b0, nb = window
    h = H(cfg)
    Xh = h.dhr(padded(pr["Y"], ((cfg.Nk + 3) // 4) * 4), s0, ns, b0, nb)
    torch.cuda.synchronize()
    Xo = oracle.dhr(pr["Y"].numpy(), cfg.Nv, cfg.Nr, cfg.Nc, slice0=s0, n_slices=ns, bin0=b0, n_bins=nb)
    assert rel(Xh, Xo) <= 1e-4, rel(Xh, Xo)


@pytest.mark.parametrize("ws_chunk_slices", [1, 3])
def test_dhr_small_workspace(H, ws_chunk_slices):
    """A workspace of a few (16-bin chunk x slice) units: hsnct_dhr runs several passes."""
    import paper_2410_22500_b200.hsnct as hm
    cfg = sd.custom(idx=21, Nc=40, Nv=16, Nr=3, Nk=70, K=2)
    pr = sd.make_problem(cfg)
    h = H(cfg)
    per_chunk = cfg.Nv * cfg.Nc * 16 * 4
    assert h.workspace_bytes(hm.OP_DHR) == per_chunk * 5  # one slice, all bins (5 chunks of 16)
    ws = torch.empty(per_chunk * ws_chunk_slices, dtype=torch.uint8, device=DEV)
    Xh = h.dhr(padded(pr["Y"], 72), 0, 3, 1, 67, ws=ws)
    torch.cuda.synchronize()
    Xo = oracle.dhr(pr["Y"].numpy(), cfg.Nv, cfg.Nr, cfg.Nc, slice0=0, n_slices=3, bin0=1, n_bins=67)
    assert rel(Xh, Xo) <= 1e-4, rel(Xh, Xo)


def test_linearity_identity_on_gpu(H):
    """Y = V D exactly: fbp + synthesize == dhr."""
    cfg = sd.custom(idx=21, Nc=40, Nv=30, Nr=2, Nk=23, K=3)
    g = torch.Generator().manual_seed(6)
    V = torch.randint(0, 8, (cfg.Np, cfg.K), generator=g).float()
    D = torch.randint(0, 8, (cfg.K, cfg.Nk), generator=g).float() / 4
    Y = (V.double() @ D.double()).float()
    h = H(cfg)
    X = h.fbp(V.to(DEV))
    a = h.synthesize(X, D.to(DEV))
    b = h.dhr(padded(Y, 24))
    torch.cuda.synchronize()
    assert rel(a, b) <= 1e-5


# ------------------------------------------------------------ whole pipeline
@pytest.mark.parametrize("cfgi,n_iter", [(1, 100), (2, 8)])
def test_fhr_pipeline_parity(H, cfgi, n_iter):
    cfg = sd.CONFIGS[cfgi]
    pr = sd.make_problem(cfg)
    h = H(cfg)
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    h.subspace_decompose(pr["Y"].to(DEV), V, D, n_iter)
    X = h.fbp(V)
    Xh = h.synthesize(X, D)
    h.sync()
    Vo, Do = oracle.nmf(pr["Y"].numpy(), pr["V0"].numpy(), pr["D0"].numpy(), n_iter)
    Xo = oracle.fbp(Vo, cfg.Nv, cfg.Nr, cfg.Nc)
    Xho = oracle.synthesize(Xo, Do)
    assert rel(Xh, Xho) <= 1e-3, rel(Xh, Xho)


def test_fhr_host_matches_device_path(H):
    cfg = sd.CONFIGS[1]
    pr = sd.make_problem(cfg)
    h = H(cfg)
    n = 25
    Vh = torch.empty_like(pr["V0"])
    Dh = torch.empty_like(pr["D0"])
    Xh_host = h.fhr_host(pr["Y"].pin_memory(), pr["V0"], pr["D0"], n, V=Vh, D=Dh)
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    h.subspace_decompose(pr["Y"].to(DEV), V, D, n)
    Xh = h.synthesize(h.fbp(V), D)
    h.sync()
    assert torch.equal(Vh, V.cpu()) and torch.equal(Dh, D.cpu())
    assert torch.equal(Xh_host, Xh.cpu())


@pytest.mark.parametrize("wsl", [1, 2, 5])
def test_fhr_stream_windows_match_device_path(H, wsl):
    """hsnct_fhr_stream: every x^h window is delivered once, in order, and equals the device
    path bit for bit (same kernels on the same inputs); ragged last window (5 slices)."""
    cfg = sd.custom(idx=41, Nc=24, Nv=12, Nr=5, Nk=72, K=3, M=3)
    pr = sd.make_problem(cfg)
    h = H(cfg)
    n = 15
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    h.subspace_decompose(pr["Y"].to(DEV), V, D, n)
    Xh = h.synthesize(h.fbp(V), D)
    h.sync()
    Xh = Xh.cpu()
    got = []
    per = cfg.Nc * cfg.Nc

    def on_window(s0, ns, xh):
        got.append((s0, ns))
        assert torch.equal(xh, Xh[s0 * per:(s0 + ns) * per])

    Vh = torch.empty_like(pr["V0"])
    h.fhr_stream(pr["Y"].pin_memory(), pr["V0"], pr["D0"], n, window_slices=wsl, on_window=on_window, V=Vh)
    assert got == [(s, min(wsl, cfg.Nr - s)) for s in range(0, cfg.Nr, wsl)]
    assert torch.equal(Vh, V.cpu())


# ----------------------------------------------------------------- errors
def test_deferred_data_errors(H):
    from paper_2410_22500_b200 import HsnctError
    cfg = sd.custom(idx=22, Nc=16, Nv=8, Nk=12, K=2)
    h = H(cfg)
    Y = torch.rand((cfg.Np, cfg.Nk), device=DEV)
    V = torch.rand((cfg.Np, 2), device=DEV) + 0.1
    D = torch.rand((2, cfg.Nk), device=DEV) + 0.1
    Y[3, 4] = float("nan")
    h.subspace_decompose(Y, V.clone(), D.clone(), 2)
    with pytest.raises(HsnctError) as e:
        h.sync()
    assert e.value.status == 2
    h.sync()  # cleared
    h.subspace_decompose(-torch.rand((cfg.Np, cfg.Nk), device=DEV), V.clone(), D.clone(), 2)
    with pytest.raises(HsnctError) as e:
        h.sync()
    assert e.value.status == 2
    Dn = D.clone()
    Dn[0, 0] = -1.0
    h.subspace_decompose(torch.rand((cfg.Np, cfg.Nk), device=DEV), V.clone(), Dn, 1)
    with pytest.raises(HsnctError) as e:
        h.sync()
    assert e.value.status == 2


def test_argument_errors(H):
    from paper_2410_22500_b200 import HsnctError
    cfg = sd.custom(idx=23, Nc=16, Nv=8, Nk=12, K=2)
    h = H(cfg)
    Y = torch.rand((cfg.Np, cfg.Nk), device=DEV)
    V = torch.rand((cfg.Np, 2), device=DEV)
    D = torch.rand((2, cfg.Nk), device=DEV)
    with pytest.raises(HsnctError):
        h.subspace_decompose(Y, V, D, -1)
    small = torch.empty(8, dtype=torch.uint8, device=DEV)
    with pytest.raises(HsnctError) as e:
        h.subspace_decompose(Y, V, D, 1, ws=small)
    assert e.value.status == 1
    with pytest.raises(HsnctError):
        h.synthesize(torch.zeros((2, 1, 16, 16), device=DEV), D, 0, 2, 0, 12)
    Ybig = torch.rand((cfg.Np, 13), device=DEV)[:, 1:]   # misaligned base
    with pytest.raises(HsnctError):
        h.subspace_decompose(Ybig, V, D, 1)
    import ctypes
    from paper_2410_22500_b200 import hsnct as hm
    ws = h.workspace(hm.OP_DECOMPOSE)
    st = hm.lib().hsnct_subspace_decompose(h._h, ctypes.c_void_p(Y.data_ptr()), 12,
                                           ctypes.c_void_p(Y.data_ptr()), ctypes.c_void_p(D.data_ptr()),
                                           1, None, ctypes.c_void_p(ws.data_ptr()), ws.numel(), None)
    assert st == 1 and b"overlap" in hm.lib().hsnct_last_error()


@pytest.mark.parametrize("plan,cfg", [
    ("ffma", sd.CONFIGS[1]),
    ("tc", sd.CONFIGS[1]),
    ("mma", sd.CONFIGS[1]),
    ("mma", sd.custom(idx=74, Nc=20, Nv=13, Nk=203, K=5, M=4)),             # ragged N_k and N_p
    ("ffma", sd.custom(idx=71, Nc=24, Nv=10, Nr=2, Nk=64, K=12, M=5)),      # K > 8 on the fused kernel
    ("twopass", sd.custom(idx=73, Nc=24, Nv=10, Nr=2, Nk=64, K=12, M=5)),   # the two-pass kernels
    ("ffma", sd.custom(idx=72, Nc=20, Nv=13, Nk=203, K=5, M=4)),            # ragged N_k (masked padding)
])
def test_clamped_count_statistic(monkeypatch, plan, cfg):
    """hsnct_decompose_stats: the number of negative Y entries clamped to 0 (reading R6) is
    exact on every row-pass plan, and counts only the N_k real bins (NaN-poisoned padding)."""
    monkeypatch.setenv("HSNCT_NMF", plan)
    from paper_2410_22500_b200 import Hsnct
    pr = sd.make_problem(cfg)
    h = Hsnct(cfg.Nv, cfg.Nr, cfg.Nc, cfg.Nk, cfg.K, device=0)
    Yd = padded(pr["Y"], ((cfg.Nk + 3) // 4) * 4 + 4, fill=-1.0)
    V = pr["V0"].to(DEV).clone()
    D = pr["D0"].to(DEV).clone()
    h.subspace_decompose(Yd, V, D, 2)
    h.sync()
    assert h.decompose_stats()["n_clamped"] == int((pr["Y"] < 0).sum())
    assert int((pr["Y"] < 0).sum()) > 0
