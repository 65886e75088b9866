"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs).

This module is the ONE piece shared by the oracle side (tests, bench's cpu
baseline) and the CUDA side (bench, GPU tests).  It holds none of the
method's arithmetic -- no NMF, no filtering, no backprojection, no subspace
expansion.  It only draws inputs:

* a phantom of N_m non-overlapping materials made of ellipses / ellipsoids
  ("a synthetic phantom x^m that contains 3 distinct,
  non-overlapping materials"), with BASELINE.json's shapes;
* mu-spectra with a 1/lambda-like baseline plus seeded Bragg-edge step drops
  (stand-in for the BEM library spectra);
* exact analytic parallel-beam line integrals of every material
  (the forward model Eq. 3, with w = 0), so
  p_true = P mu^T is exactly rank N_m;
* Poisson counts for the open beam and the sample (Eq. 10 and PAPER.md:390-396)
  and the -log transform Eq. 2 with a 1/2-count floor
  (reading R7) through a 256-entry fp64 log table;
* the strictly positive NMF initialisation (reading R4).

Recipe constants are proposals (DESIGN.md §4 "Inputs"); the paper gives none.
Geometry conventions (R13, R14): theta_v = v*pi/N_v; detector
coordinate t_c = c - (N_c-1)/2; voxel (i, j) at x = j-(N_c-1)/2,
y = i-(N_c-1)/2; a ray at (theta, t) is {x cos(theta) + y sin(theta) = t}.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np
import torch


@dataclass(frozen=True)
class Config:
    idx: int            # BASELINE.json configs[idx-1]
    Nc: int             # detector columns = image width
    Nr: int             # detector rows = slices
    Nv: int             # views over 180 degrees
    Nk: int             # wavelength bins on [1, 5] Angstrom
    K: int              # subspace dimension N_s
    n_iter: int         # NMF iterations (R5, R21)
    M: int              # materials N_m
    counts: float       # open-beam mean counts per bin
    close_edges: bool   # two materials with Bragg edges 3 bins apart

    @property
    def Np(self) -> int:
        return self.Nv * self.Nr * self.Nc

    @property
    def Nx(self) -> int:
        return self.Nr * self.Nc * self.Nc

    @property
    def name(self) -> str:
        return f"C{self.idx}"

    def describe(self) -> str:
        return (f"C{self.idx}: Nc={self.Nc} Nr={self.Nr} Nv={self.Nv} Nk={self.Nk} K={self.K} "
                f"iters={self.n_iter} M={self.M} counts={self.counts:g}")


CONFIGS = {
    1: Config(1, 64, 1, 90, 200, 3, 100, 3, 100.0, False),
    2: Config(2, 256, 1, 180, 1200, 4, 200, 4, 50.0, False),
    3: Config(3, 256, 64, 120, 1600, 5, 200, 5, 30.0, False),
    4: Config(4, 512, 128, 64, 1600, 6, 300, 6, 20.0, True),
    5: Config(5, 512, 256, 64, 1600, 6, 300, 6, 20.0, True),
    # not in BASELINE.json: the paper's Table I simulated-data shape:
    # 512 x 512 detector, N_r = 512 slices, N_v = 32 views, N_k = 1200, N_s = 9 (K > 8)
    6: Config(6, 512, 512, 32, 1200, 9, 300, 3, 20.0, False),
}


def custom(**kw) -> Config:
    """A config with explicit shapes (ragged / edge-case tests)."""
    base = dict(idx=0, Nc=16, Nr=1, Nv=8, Nk=12, K=2, n_iter=5, M=2, counts=100.0,
                close_edges=False)
    base.update(kw)
    return Config(**base)


def reduced(cfg: Config, Nr: int) -> Config:
    """Slice-reduced variant (same N_v, N_c, N_k, K, iterations, counts)."""
    return replace(cfg, Nr=Nr)


def seeds(cfg: Config):
    c = cfg.idx
    return dict(phantom=1000 * c + 1, spectra=1000 * c + 2, noise=1000 * c + 3, init=1000 * c + 4)


def wavelengths(Nk: int) -> np.ndarray:
    """Bin centres lambda_k = 1 + 4 (k + 1/2) / N_k Angstrom (R18)."""
    return 1.0 + 4.0 * (np.arange(Nk) + 0.5) / Nk


def view_angles(Nv: int) -> np.ndarray:
    """theta_v = v pi / N_v, endpoint excluded (R13)."""
    return np.arange(Nv) * math.pi / Nv


# --------------------------------------------------------------------------
# Phantom: ellipses (2D) / ellipsoids (3D), non-overlapping in plane.
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Ellipsoid:
    material: int
    x0: float
    y0: float
    z0: float
    a: float      # in-plane semi-axis along the rotated x'
    b: float      # in-plane semi-axis along the rotated y'
    c: float      # z semi-axis (inf for 2D)
    alpha: float  # in-plane rotation


def make_phantom(cfg: Config, seed: int | None = None):
    """1-2 ellipses per material; disjoint bounding circles + 1 px."""
    rng = np.random.default_rng(seeds(cfg)["phantom"] if seed is None else seed)
    Nc, Nr = cfg.Nc, cfg.Nr
    shapes: list[Ellipsoid] = []
    placed: list[tuple[float, float, float]] = []
    for m in range(cfg.M):
        n_shapes = int(rng.integers(1, 3))
        got = 0
        for _ in range(4000):
            if got == n_shapes:
                break
            a = rng.uniform(0.05, 0.12) * Nc
            b = rng.uniform(0.05, 0.12) * Nc
            R = max(a, b)
            rho_max = min(0.38 * Nc, 0.47 * Nc - R)
            rho = rho_max * math.sqrt(rng.uniform())
            phi = rng.uniform(0, 2 * math.pi)
            x0, y0 = rho * math.cos(phi), rho * math.sin(phi)
            if any(math.hypot(x0 - px, y0 - py) < R + pr + 1.0 for px, py, pr in placed):
                continue
            alpha = rng.uniform(0, math.pi)
            if Nr > 1:
                z0 = rng.uniform(-0.25, 0.25) * Nr
                cz = rng.uniform(0.3, 0.5) * Nr
            else:
                z0, cz = 0.0, math.inf
            shapes.append(Ellipsoid(m, x0, y0, z0, a, b, cz, alpha))
            placed.append((x0, y0, R))
            got += 1
        if got == 0:
            raise RuntimeError("phantom: could not place material %d" % m)
    return shapes


def _slice_scale(e: Ellipsoid, z: float) -> float:
    if math.isinf(e.c):
        return 1.0
    t = (z - e.z0) / e.c
    return math.sqrt(1.0 - t * t) if abs(t) < 1.0 else 0.0


def slice_z(Nr: int) -> np.ndarray:
    return np.arange(Nr) - 0.5 * (Nr - 1)


def rasterize(shapes, cfg: Config, r: int, supersample: int = 1) -> np.ndarray:
    """Volume fractions x^m of slice r: [M, Nc, Nc] (diagnostics and pins only)."""
    Nc = cfg.Nc
    z = slice_z(cfg.Nr)[r]
    s = supersample
    off = (np.arange(s) + 0.5) / s - 0.5
    ii = (np.arange(Nc)[:, None] + off[None, :]).reshape(-1) - 0.5 * (Nc - 1)
    y = ii[:, None] * np.ones((1, Nc * s))
    x = np.ones((Nc * s, 1)) * ii[None, :]
    out = np.zeros((cfg.M, Nc, Nc))
    for e in shapes:
        f = _slice_scale(e, z)
        if f <= 0:
            continue
        ca, sa = math.cos(e.alpha), math.sin(e.alpha)
        xr = (x - e.x0) * ca + (y - e.y0) * sa
        yr = -(x - e.x0) * sa + (y - e.y0) * ca
        inside = (xr / (e.a * f)) ** 2 + (yr / (e.b * f)) ** 2 <= 1.0
        out[e.material] += inside.reshape(Nc, s, Nc, s).mean(axis=(1, 3))
    return out


def ellipse_line_integrals(theta: torch.Tensor, t: torch.Tensor, x0, y0, a, b, alpha, mu=1.0):
    """Exact parallel-beam line integral of a uniform ellipse (Kak & Slaney ch. 3):
    P(theta, t) = 2 mu a b sqrt(a2 - s^2) / a2 for s^2 <= a2, else 0, with
    s = t - (x0 cos theta + y0 sin theta), a2 = a^2 cos^2(theta-alpha) + b^2 sin^2(theta-alpha).
    Broadcasts over theta and t (fp64)."""
    s = t - (x0 * torch.cos(theta) + y0 * torch.sin(theta))
    a2 = (a * torch.cos(theta - alpha)) ** 2 + (b * torch.sin(theta - alpha)) ** 2
    inside = (a2 - s * s).clamp_min(0.0)
    return 2.0 * mu * a * b * torch.sqrt(inside) / a2


def material_sinograms(shapes, cfg: Config, device="cpu") -> torch.Tensor:
    """P[m, v, r, c] fp64: exact line integrals of every material's volume fraction."""
    Nv, Nr, Nc = cfg.Nv, cfg.Nr, cfg.Nc
    theta = torch.as_tensor(view_angles(Nv), dtype=torch.float64, device=device)[:, None]
    t = (torch.arange(Nc, dtype=torch.float64, device=device) - 0.5 * (Nc - 1))[None, :]
    P = torch.zeros((cfg.M, Nv, Nr, Nc), dtype=torch.float64, device=device)
    zs = slice_z(Nr)
    for e in shapes:
        for r in range(Nr):
            f = _slice_scale(e, float(zs[r]))
            if f <= 0:
                continue
            P[e.material, :, r, :] += ellipse_line_integrals(theta, t, e.x0, e.y0, e.a * f,
                                                             e.b * f, e.alpha)
    return P


# --------------------------------------------------------------------------
# Spectra: 1/lambda-like baseline + Bragg-edge step drops.
# --------------------------------------------------------------------------

def make_spectra(cfg: Config, seed: int | None = None) -> np.ndarray:
    """mu_m(lambda_k) = a_m + b_m/lambda + sum_e J_{m,e} [lambda < lambda_{m,e}]  -> [M, Nk]."""
    rng = np.random.default_rng(seeds(cfg)["spectra"] if seed is None else seed)
    lam = wavelengths(cfg.Nk)
    mu = np.zeros((cfg.M, cfg.Nk))
    edges = []
    for m in range(cfg.M):
        a = rng.uniform(0.2, 0.6)
        b = rng.uniform(0.2, 1.0)
        E = int(rng.integers(3, 6))
        le = rng.uniform(1.2, 4.8, size=E)
        J = rng.uniform(0.1, 0.4, size=E) * (a + b)
        edges.append((le, J))
        mu[m] = a + b / lam
    if cfg.close_edges and cfg.M >= 2:
        # "two with closely spaced Bragg edges": materials 0 and 1 share an edge pair
        # 3 bins apart (3 * 4/N_k Angstrom).
        base = edges[0][0][0]
        le1 = edges[1][0].copy()
        le1[0] = base + 3 * 4.0 / cfg.Nk
        edges[1] = (le1, edges[1][1])
    for m, (le, J) in enumerate(edges):
        for e in range(len(le)):
            mu[m] += J[e] * (lam < le[e])
    return mu


# --------------------------------------------------------------------------
# Counts and -log projections.
# --------------------------------------------------------------------------

def log_table() -> np.ndarray:
    """L[n] = ln(max(n, 1/2)), n = 0..255, fp64 (R7)."""
    n = np.arange(256, dtype=np.float64)
    return np.log(np.maximum(n, 0.5))


def expected_counts(ptrue: torch.Tensor, counts: float) -> torch.Tensor:
    """Mean transmitted counts C exp(-p) (Eq. 10 without noise), fp64."""
    return counts * torch.exp(-ptrue)


def neglog(y0: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    """Eq. 2 on (possibly real-valued) counts with the 1/2-count floor (R7):
    ln(max(y0, 1/2)) - ln(max(y, 1/2)), fp64.  The integer-count path in make_problem uses the
    same function through the 256-entry table log_table()."""
    return torch.log(torch.clamp(y0.double(), min=0.5)) - torch.log(torch.clamp(y.double(), min=0.5))


def make_problem(cfg: Config, device="cpu", noise: bool = True, chunk_rows: int = 1 << 18,
                 dtype_y=torch.float32, return_counts: bool = False):
    """Draw (Y, V0, D0) for a config.  Returns a dict:

    Y   [Np, Nk] fp32, -log transmission (Eq. 2), row p = (v Nr + r) Nc + c.
    V0  [Np, K]  fp32 > 0,  D0 [K, Nk] fp32 > 0 (reading R4).
    P   [M, Nv, Nr, Nc] fp64 material sinograms, mu [M, Nk] fp64 spectra (scaled),
    shapes, angles, plus the config.
    With noise=False, Y = fp32(p_true): exactly rank M in fp64 before the cast.
    return_counts=True adds the uint8 counts: y0 [Nr*Nc, Nk] (open beam, shared by all
    views) and y [Np, Nk], with Y[p] = fp32(L[y0[p % (Nr*Nc)]] - L[y[p]]) (noise=True only).
    """
    dev = torch.device(device)
    shapes = make_phantom(cfg)
    P = material_sinograms(shapes, cfg, device=dev)                   # [M,Nv,Nr,Nc]
    mu = make_spectra(cfg)                                            # [M,Nk]
    pmax = float((P.reshape(cfg.M, -1) * torch.as_tensor(mu.max(axis=1), device=dev,
                                                          dtype=torch.float64)[:, None]).sum(0).max())
    scale = 1.5 / pmax if pmax > 0 else 1.0
    mu = mu * scale
    mu_t = torch.as_tensor(mu, dtype=torch.float64, device=dev)
    Pm = P.reshape(cfg.M, cfg.Np).T.contiguous()                      # [Np, M]
    Y = torch.empty((cfg.Np, cfg.Nk), dtype=dtype_y, device=dev)
    L = torch.as_tensor(log_table(), dtype=torch.float64, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(seeds(cfg)["noise"])
    if noise:
        # open beam y°_{r,c,k} ~ Poisson(C), shared by all views
        ob = torch.poisson(torch.full((cfg.Nr * cfg.Nc, cfg.Nk), float(cfg.counts),
                                      dtype=torch.float64, device=dev), generator=g)
        assert float(ob.max()) <= 255.0
        Lob = L[ob.long()]
        if return_counts:
            y_all = torch.empty((cfg.Np, cfg.Nk), dtype=torch.uint8, device=dev)
    for p0 in range(0, cfg.Np, chunk_rows):
        p1 = min(cfg.Np, p0 + chunk_rows)
        ptrue = Pm[p0:p1] @ mu_t                                      # Eq. 3, w = 0
        if noise:
            y = torch.poisson(expected_counts(ptrue, cfg.counts), generator=g)   # Eq. 10 + Poisson
            assert float(y.max()) <= 255.0
            if return_counts:
                y_all[p0:p1] = y.to(torch.uint8)
            rc = torch.arange(p0, p1, device=dev) % (cfg.Nr * cfg.Nc)
            Y[p0:p1] = (Lob[rc] - L[y.long()]).to(dtype_y)            # Eq. 2 via the log table
        else:
            Y[p0:p1] = ptrue.to(dtype_y)
    V0, D0 = make_init(Y, cfg.K, seeds(cfg)["init"])
    out = dict(cfg=cfg, Y=Y, V0=V0, D0=D0, P=P, mu=mu, shapes=shapes, angles=view_angles(cfg.Nv))
    if return_counts and noise:
        out["y0"] = ob.to(torch.uint8)
        out["y"] = y_all
    return out


def make_init(Y: torch.Tensor, K: int, seed: int):
    """s = sqrt(mean(Y+)/K); V0 = s (1-U), D0 = s (1-U), U ~ U[0,1): strictly positive (R4)."""
    g = torch.Generator(device=Y.device)
    g.manual_seed(seed)
    Np, Nk = Y.shape
    tot = 0.0  # mean(Y+) in fp64, accumulated over row chunks (no full-size fp64 copy of Y)
    for p0 in range(0, Np, 1 << 18):
        tot += float(Y[p0:p0 + (1 << 18)].clamp_min(0).sum(dtype=torch.float64))
    s = math.sqrt(max(tot / (Np * Nk), 1e-12) / K)
    V0 = (s * (1.0 - torch.rand((Np, K), generator=g, device=Y.device, dtype=torch.float64))).float()
    D0 = (s * (1.0 - torch.rand((K, Nk), generator=g, device=Y.device, dtype=torch.float64))).float()
    return V0, D0


def random_lowrank(Np: int, Nk: int, K: int, seed: int, device="cpu"):
    """Y = V* D* exactly in fp64 (then fp32), with V*, D* > 0 (fixed-point / identity pins)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    Vs = torch.rand((Np, K), generator=g, device=device, dtype=torch.float64) + 0.1
    Ds = torch.rand((K, Nk), generator=g, device=device, dtype=torch.float64) + 0.1
    return Vs, Ds


def region_labels(pr, slices=None) -> np.ndarray:
    """User-provided homogeneous regions for FMD's semi-supervised mode (Algorithm 2 input M,
    PAPER.md:276-278): label m where the phantom voxel is pure material m (volume fraction 1),
    -1 elsewhere.  int32 [Nr, Nc, Nc] (or the given slices)."""
    cfg = pr["cfg"]
    rs = range(cfg.Nr) if slices is None else slices
    out = []
    for r in rs:
        f = rasterize(pr["shapes"], cfg, r)
        lab = np.full((cfg.Nc, cfg.Nc), -1, np.int32)
        for m in range(cfg.M):
            lab[f[m] >= 1.0] = m
        out.append(lab)
    return np.stack(out)
