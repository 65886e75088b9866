"""CPU fp64 oracle for the FHR hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2410_22500_b200``) never imports it and has no CPU fallback.

This module is argument marshalling (numpy <-> C) around ``oracle/oracle.c``;
every formula lives in the C file with its PAPER.md citation.  The shared
library is compiled on first use (``gcc -O2 -fopenmp``, no ``-ffast-math``)
if ``__graft_entry__.build()`` has not already built it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_f64p = ctypes.POINTER(ctypes.c_double)
_f32p = ctypes.POINTER(ctypes.c_float)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64
_int = ctypes.c_int


def build(force: bool = False) -> str:
    """Compile oracle/oracle.c into oracle/liboracle.so (plain gcc, fp64)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            L.oracle_max_threads.restype = _int
            L.oracle_nmf_objective.restype = ctypes.c_double
            L.oracle_nmf_objective.argtypes = [_f32p, _i64, _i64, _i64, _int, _f64p, _f64p, _int]
            L.oracle_nmf.restype = _int
            L.oracle_nmf.argtypes = [_f32p, _i64, _i64, _i64, _int, _f64p, _f64p, _int, _f64p, _int]
            L.oracle_nmf_vstep_rows.restype = _int
            L.oracle_nmf_vstep_rows.argtypes = [_f32p, _i64, _i64, _i64, _int, _f64p, _f64p,
                                                _i64p, _i64, _f64p, _int]
            L.oracle_nmf_dstep_cols.restype = _int
            L.oracle_nmf_dstep_cols.argtypes = [_f32p, _i64, _i64, _i64, _int, _f64p, _f64p,
                                                _i64p, _i64, _f64p, _int]
            L.oracle_ramp_kernel.restype = ctypes.c_double
            L.oracle_ramp_kernel.argtypes = [_i64]
            L.oracle_ramp_filter_rows.restype = None
            L.oracle_ramp_filter_rows.argtypes = [_f64p, _f64p, _i64, _i64, _int]
            L.oracle_backproject_slice.restype = None
            L.oracle_backproject_slice.argtypes = [_f64p, _i64, _i64, _f64p, _f64p]
            L.oracle_splat_project_slice.restype = None
            L.oracle_splat_project_slice.argtypes = [_f64p, _i64, _i64, _f64p, _f64p]
            L.oracle_qggmrf_rho.restype = ctypes.c_double
            L.oracle_qggmrf_rho.argtypes = [ctypes.c_double, _f64p]
            L.oracle_qggmrf_omega.restype = ctypes.c_double
            L.oracle_qggmrf_omega.argtypes = [ctypes.c_double, _f64p]
            L.oracle_mbir_project_slice.restype = None
            L.oracle_mbir_project_slice.argtypes = [_f64p, _i64, _i64, _f64p, _f64p]
            L.oracle_mbir_backproject_slice.restype = None
            L.oracle_mbir_backproject_slice.argtypes = [_f64p, _i64, _i64, _f64p, _f64p]
            L.oracle_mbir_slice.restype = _int
            L.oracle_mbir_slice.argtypes = [_f64p, _i64, _i64, _f64p, _f64p, _int, _f64p, _f64p]
            L.oracle_mbir.restype = _int
            L.oracle_mbir.argtypes = [_f64p, _i64, _i64, _i64, _int, _f64p, _f64p, _int, _f64p, _int]
            L.oracle_radon_naive.restype = None
            L.oracle_radon_naive.argtypes = [_f64p, _i64, _i64, _f64p, ctypes.c_double, _f64p, _int]
            L.oracle_fbp.restype = _int
            L.oracle_fbp.argtypes = [_f64p, _i64, _i64, _i64, _int, _f64p, _f64p, _int]
            L.oracle_synthesize.restype = _int
            L.oracle_synthesize.argtypes = [_f64p, _f64p, _i64, _i64, _i64, _int, _i64, _i64,
                                            _i64, _i64, _f64p, _int]
            L.oracle_fmd_transform.restype = _int
            L.oracle_fmd_transform.argtypes = [_f64p, _i64, _int, ctypes.POINTER(ctypes.c_int32), _int, _f64p,
                                               _i64p]
            L.oracle_nnls.restype = _int
            L.oracle_nnls.argtypes = [_f64p, _int, _int, _f64p, _f64p]
            L.oracle_fmd_materials.restype = ctypes.c_int64
            L.oracle_fmd_materials.argtypes = [_f64p, _i64, _int, _f64p, _int, _f64p, _int]
            L.oracle_counts_to_projections.restype = None
            L.oracle_counts_to_projections.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, _i64, _i64,
                                                       _i64, _f64p]
            L.oracle_fmd_spectra.restype = None
            L.oracle_fmd_spectra.argtypes = [_f64p, _i64, _int, _f64p, _int, _f64p]
            L.oracle_dhr.restype = _int
            L.oracle_dhr.argtypes = [_f32p, _i64, _i64, _i64, _i64, _i64, _f64p, _i64, _i64,
                                     _i64, _i64, _f64p, _int]
            _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _p64(a):
    return a.ctypes.data_as(_f64p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _y32(Y):
    Y = np.asarray(Y)
    if Y.dtype != np.float32 or Y.ndim != 2 or Y.strides[1] != 4 or Y.strides[0] % 4:
        Y = np.ascontiguousarray(Y, dtype=np.float32)
    return Y, Y.strides[0] // 4


def _angles(angles):
    if angles is None:
        return None, None
    a = _f64(angles)
    return a, _p64(a)


def nmf(Y, V0, D0, n_iter, objective=False, nthreads=0):
    """Lee-Seung NMF trajectory (oracle.c: oracle_nmf).  Returns (V, D[, obj])."""
    Y, ld = _y32(Y)
    Np, Nk = Y.shape
    V = _f64(V0).copy()
    D = _f64(D0).copy()
    K = V.shape[1]
    assert V.shape == (Np, K) and D.shape == (K, Nk)
    obj = np.zeros(2 * n_iter) if objective else None
    rc = lib().oracle_nmf(Y.ctypes.data_as(_f32p), Np, Nk, ld, K, _p64(V), _p64(D), int(n_iter),
                          _p64(obj) if objective else None, int(nthreads))
    if rc:
        raise ValueError("oracle_nmf: bad arguments")
    return (V, D, obj) if objective else (V, D)


def nmf_objective(Y, V, D, nthreads=0):
    Y, ld = _y32(Y)
    V = _f64(V)
    D = _f64(D)
    return float(lib().oracle_nmf_objective(Y.ctypes.data_as(_f32p), Y.shape[0], Y.shape[1], ld,
                                            V.shape[1], _p64(V), _p64(D), int(nthreads)))


def nmf_vstep_rows(Y, V, D, rows, nthreads=0):
    Y, ld = _y32(Y)
    V = _f64(V)
    D = _f64(D)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    K = V.shape[1]
    out = np.zeros((rows.size, K))
    lib().oracle_nmf_vstep_rows(Y.ctypes.data_as(_f32p), Y.shape[0], Y.shape[1], ld, K, _p64(V),
                                _p64(D), rows.ctypes.data_as(_i64p), rows.size, _p64(out),
                                int(nthreads))
    return out


def nmf_dstep_cols(Y, V, D, cols, nthreads=0):
    Y, ld = _y32(Y)
    V = _f64(V)
    D = _f64(D)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    K = V.shape[1]
    out = np.zeros((K, cols.size))
    lib().oracle_nmf_dstep_cols(Y.ctypes.data_as(_f32p), Y.shape[0], Y.shape[1], ld, K, _p64(V),
                                _p64(D), cols.ctypes.data_as(_i64p), cols.size, _p64(out),
                                int(nthreads))
    return out


def ramp_kernel(d: int) -> float:
    return float(lib().oracle_ramp_kernel(int(d)))


def ramp_filter_rows(S, nthreads=0):
    S = _f64(S)
    nc = S.shape[-1]
    Q = np.zeros_like(S)
    lib().oracle_ramp_filter_rows(_p64(S), _p64(Q), S.size // nc if nc else 0, nc, int(nthreads))
    return Q


def backproject_slice(Q, angles=None):
    """Q: [Nv, Nc] filtered sinogram of one slice -> X [Nc, Nc]."""
    Q = _f64(Q)
    nv, nc = Q.shape
    a, ap = _angles(angles)
    X = np.zeros((nc, nc))
    lib().oracle_backproject_slice(_p64(Q), nv, nc, ap, _p64(X))
    return X


def splat_project_slice(X, nv, angles=None):
    X = _f64(X)
    nc = X.shape[0]
    a, ap = _angles(angles)
    P = np.zeros((nv, nc))
    lib().oracle_splat_project_slice(_p64(X), nv, nc, ap, _p64(P))
    return P


def radon_naive(img, nv, angles=None, step=0.25, nthreads=0):
    img = _f64(img)
    nc = img.shape[0]
    a, ap = _angles(angles)
    P = np.zeros((nv, nc))
    lib().oracle_radon_naive(_p64(img), nc, nv, ap, float(step), _p64(P), int(nthreads))
    return P


def fbp(V, Nv, Nr, Nc, angles=None, nthreads=0):
    """V: [Np, K] subspace views -> X [K, Nr, Nc, Nc]."""
    V = _f64(V)
    K = V.shape[1]
    assert V.shape[0] == Nv * Nr * Nc
    a, ap = _angles(angles)
    X = np.zeros((K, Nr, Nc, Nc))
    if lib().oracle_fbp(_p64(V), Nv, Nr, Nc, K, ap, _p64(X), int(nthreads)):
        raise ValueError("oracle_fbp: bad arguments")
    return X


def synthesize(X, D, slice0=0, n_slices=None, bin0=0, n_bins=None, nthreads=0):
    """X: [K, Nr, Nc, Nc], D: [K, Nk] -> Xh [n_slices*Nc*Nc, n_bins]."""
    X = _f64(X)
    D = _f64(D)
    K, Nr, Nc, _ = X.shape
    Nk = D.shape[1]
    n_slices = Nr - slice0 if n_slices is None else n_slices
    n_bins = Nk - bin0 if n_bins is None else n_bins
    Xh = np.zeros((n_slices * Nc * Nc, n_bins))
    if lib().oracle_synthesize(_p64(X), _p64(D), Nr, Nc, Nk, K, slice0, n_slices, bin0, n_bins,
                               _p64(Xh), int(nthreads)):
        raise ValueError("oracle_synthesize: bad window")
    return Xh


def dhr(Y, Nv, Nr, Nc, angles=None, slice0=0, n_slices=None, bin0=0, n_bins=None, nthreads=0):
    """Per-bin FBP of Y [Np, Nk] -> Xh [n_slices*Nc*Nc, n_bins]."""
    Y, ld = _y32(Y)
    Nk = Y.shape[1]
    n_slices = Nr - slice0 if n_slices is None else n_slices
    n_bins = Nk - bin0 if n_bins is None else n_bins
    a, ap = _angles(angles)
    Xh = np.zeros((n_slices * Nc * Nc, n_bins))
    if lib().oracle_dhr(Y.ctypes.data_as(_f32p), ld, Nv, Nr, Nc, Nk, ap, slice0, n_slices, bin0,
                        n_bins, _p64(Xh), int(nthreads)):
        raise ValueError("oracle_dhr: bad window")
    return Xh


# ------------------------------------------------------------------ FMD (NEXT-2)
def fmd_transform(X, labels, n_mat):
    """Eq. 7: T [Nm, K] region means of X [K, ...] (labels < 0: no region); counts [Nm]."""
    X = _f64(X)
    K = X.shape[0]
    X2 = np.ascontiguousarray(X.reshape(K, -1))
    Nx = X2.shape[1]
    lab = np.ascontiguousarray(np.asarray(labels).reshape(-1), dtype=np.int32)
    assert lab.size == Nx
    T = np.zeros((n_mat, K))
    counts = np.zeros(n_mat, dtype=np.int64)
    rc = lib().oracle_fmd_transform(_p64(X2), Nx, K, lab.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                    int(n_mat), _p64(T), counts.ctypes.data_as(_i64p))
    if rc == 1:
        raise ValueError("fmd_transform: label out of range")
    if rc == 2:
        raise ValueError("fmd_transform: empty region")
    return T, counts


def nnls(A, y):
    """Lawson-Hanson NNLS (oracle.c: oracle_nnls): argmin_{x>=0} ||A x - y||."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    rows, m = A.shape
    x = np.zeros(m)
    it = lib().oracle_nnls(_p64(A), rows, m, _p64(y), _p64(x))
    if it < 0:
        raise ValueError("nnls failed")
    return x


def fmd_materials(X, T, nthreads=0):
    """Eq. 8: Xm [Nm, ...] = per-voxel NNLS of X [K, ...] against T [Nm, K]."""
    X = _f64(X)
    T = _f64(T)
    K = X.shape[0]
    X2 = np.ascontiguousarray(X.reshape(K, -1))
    Nm = T.shape[0]
    Xm = np.zeros((Nm, X2.shape[1]))
    fails = lib().oracle_fmd_materials(_p64(X2), X2.shape[1], K, _p64(T), Nm, _p64(Xm), int(nthreads))
    if fails:
        raise ValueError(f"fmd_materials: NNLS failed on {fails} voxels")
    return Xm.reshape((Nm,) + X.shape[1:])


def fmd_spectra(D, T):
    """Eq. 9: (D^m)^T [Nm, Nk] = T [Nm, K] D [K, Nk]."""
    D = _f64(D)
    T = _f64(T)
    Dm = np.zeros((T.shape[0], D.shape[1]))
    lib().oracle_fmd_spectra(_p64(D), D.shape[1], D.shape[0], _p64(T), T.shape[0], _p64(Dm))
    return Dm


# ------------------------------------------------------------------ MBIR (NEXT-3)
def mbir_params(sigma_v, sigma_x, p=1.2, q=2.0, T=1.0):
    """{sv, sx, p, q, T} of oracle.c's Eq. 5 objective (R24-R26)."""
    return np.array([sigma_v, sigma_x, p, q, T], dtype=np.float64)


def qggmrf_rho(d, prm):
    return float(lib().oracle_qggmrf_rho(float(d), _p64(np.asarray(prm, np.float64))))


def qggmrf_omega(d, prm):
    return float(lib().oracle_qggmrf_omega(float(d), _p64(np.asarray(prm, np.float64))))


def mbir_project_slice(X, nv, angles=None):
    """(A x)[v][c] = sum_ij x_ij max(0, 1 - |u_ij(v) - c|) -> [nv, Nc]."""
    X = _f64(X)
    nc = X.shape[0]
    a, ap = _angles(angles)
    P = np.zeros((nv, nc))
    lib().oracle_mbir_project_slice(_p64(X), nv, nc, ap, _p64(P))
    return P


def mbir_backproject_slice(R, angles=None):
    """A^T r -> [Nc, Nc]."""
    R = _f64(R)
    nv, nc = R.shape
    a, ap = _angles(angles)
    X = np.zeros((nc, nc))
    lib().oracle_mbir_backproject_slice(_p64(R), nv, nc, ap, _p64(X))
    return X


def mbir_slice(y, x0, prm, n_iter, angles=None, objective=False):
    """SQS iterations of Eq. 5 on one slice: y [Nv, Nc], x0 [Nc, Nc] -> x (and the objective
    of iterates 0..n_iter)."""
    y = _f64(y)
    nv, nc = y.shape
    x = _f64(x0).copy()
    a, ap = _angles(angles)
    obj = np.zeros(n_iter + 1) if objective else None
    rc = lib().oracle_mbir_slice(_p64(y), nv, nc, ap, _p64(np.asarray(prm, np.float64)), int(n_iter), _p64(x),
                                 _p64(obj) if objective else None)
    if rc:
        raise ValueError("oracle_mbir_slice: bad parameters (q must be 2, p in [1, 2], sv, sx, T > 0)")
    return (x, obj) if objective else x


def mbir(V, Nv, Nr, Nc, X0, prm, n_iter, angles=None, nthreads=0):
    """V [Np, K] subspace views, X0 [K, Nr, Nc, Nc] -> X after n_iter SQS iterations per channel/slice."""
    V = _f64(V)
    K = V.shape[1]
    X = _f64(X0).copy()
    a, ap = _angles(angles)
    if lib().oracle_mbir(_p64(V), Nv, Nr, Nc, K, ap, _p64(np.asarray(prm, np.float64)), int(n_iter), _p64(X),
                         int(nthreads)):
        raise ValueError("oracle_mbir: bad parameters")
    return X


def counts_to_projections(y, y0, Nv, b=None):
    """Eq. 2 + Appendix A (oracle.c): uint8 y [Np, Nk], y0 [Nr*Nc, Nk], b [Nv, Nk] or None -> p fp64."""
    y = np.ascontiguousarray(y, dtype=np.uint8)
    y0 = np.ascontiguousarray(y0, dtype=np.uint8)
    Np, Nk = y.shape
    NrNc = y0.shape[0]
    assert Np == Nv * NrNc and y0.shape[1] == Nk
    bb = None if b is None else _f64(b).reshape(Nv, Nk)
    P = np.zeros((Np, Nk))
    lib().oracle_counts_to_projections(y.ctypes.data, y0.ctypes.data, None if bb is None else bb.ctypes.data,
                                       Nv, NrNc, Nk, _p64(P))
    return P
