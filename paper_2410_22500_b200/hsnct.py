"""Thin Python binding of libhsnct.so (include/hsnct.h) -- argument marshalling only.

PyTorch provides device memory and the current CUDA stream; every step of the
hot path runs in the library's CUDA kernels.  There is no CPU fallback: if the
shared library is missing or no CUDA device is present, construction raises.
Method names follow the C ABI (hsnct_subspace_decompose -> subspace_decompose).
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# HSNCT_LIB selects an experimental build variant (paper_2410_22500_b200/build.py --variant=...)
LIB_PATH = os.environ.get("HSNCT_LIB") or os.path.join(_HERE, "libhsnct.so")

OK, E_ARG, E_DATA, E_NUMERIC, E_CUDA, E_NOMEM = range(6)
OP_DECOMPOSE, OP_FBP, OP_DHR, OP_FHR_HOST, OP_FMD, OP_MBIR, OP_PROJECT, OP_DECOMPOSE_COUNTS = range(8)
MAX_SUB = 16

# hsnct_window_fn: void (*)(void* user, int slice0, int n_slices, const float* xh)
WINDOW_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p)

_lock = threading.Lock()
_lib = None


class HsnctError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[{status}] {message}")
        self.status = status


class _Geom(ctypes.Structure):
    _fields_ = [("n_views", ctypes.c_int32), ("n_rows", ctypes.c_int32),
                ("n_cols", ctypes.c_int32), ("n_bins", ctypes.c_int32),
                ("n_sub", ctypes.c_int32), ("angles", ctypes.POINTER(ctypes.c_double))]


class MbirParams(ctypes.Structure):
    """hsnct_mbir_params: Eq. 5 noise scale sigma_v and QGGMRF (sigma_x, p, q, T)."""
    _fields_ = [("sigma_v", ctypes.c_double), ("sigma_x", ctypes.c_double), ("p", ctypes.c_double),
                ("q", ctypes.c_double), ("T", ctypes.c_double)]


def lib():
    """Load libhsnct.so (fails loudly if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                  "(nvcc, sm_100a); there is no CPU fallback")
            L = ctypes.CDLL(LIB_PATH)
            vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
            L.hsnct_create.argtypes = [ctypes.POINTER(_Geom), i32, ctypes.POINTER(vp)]
            L.hsnct_create.restype = i32
            L.hsnct_destroy.argtypes = [vp]
            L.hsnct_destroy.restype = None
            L.hsnct_workspace_bytes.argtypes = [vp, i32]
            L.hsnct_workspace_bytes.restype = sz
            L.hsnct_subspace_decompose.argtypes = [vp, vp, i64, vp, vp, i32, vp, vp, sz, vp]
            L.hsnct_subspace_decompose.restype = i32
            L.hsnct_fbp.argtypes = [vp, vp, vp, vp, sz, vp]
            L.hsnct_mbir.argtypes = [vp, vp, vp, i32, ctypes.POINTER(MbirParams), vp, vp, sz, vp]
            L.hsnct_mbir.restype = i32
            L.hsnct_project.argtypes = [vp, vp, vp, vp, sz, vp]
            L.hsnct_counts_to_projections.argtypes = [vp, vp, vp, vp, vp, i64, vp]
            L.hsnct_counts_to_projections.restype = i32
            L.hsnct_subspace_decompose_counts.argtypes = [vp, vp, vp, vp, vp, vp, i32, vp, vp, sz, vp]
            L.hsnct_subspace_decompose_counts.restype = i32
            L.hsnct_project.restype = i32
            L.hsnct_fbp.restype = i32
            L.hsnct_synthesize.argtypes = [vp, vp, vp, i32, i32, i32, i32, vp, i64, vp]
            L.hsnct_synthesize.restype = i32
            L.hsnct_dhr.argtypes = [vp, vp, i64, i32, i32, i32, i32, vp, i64, vp, sz, vp]
            L.hsnct_dhr.restype = i32
            L.hsnct_fhr_host.argtypes = [vp, vp, i64, vp, vp, i32, vp, vp, vp, vp, sz, vp]
            L.hsnct_fhr_host.restype = i32
            L.hsnct_fhr_stream_bytes.argtypes = [vp, i32]
            L.hsnct_fhr_stream_bytes.restype = sz
            L.hsnct_fhr_stream.argtypes = [vp, vp, i64, vp, vp, i32, i32, vp, WINDOW_FN, vp, vp, vp, vp, sz, vp]
            L.hsnct_fhr_stream.restype = i32
            L.hsnct_fhr_stream_counts_bytes.argtypes = [vp, i32]
            L.hsnct_fhr_stream_counts_bytes.restype = sz
            L.hsnct_fhr_stream_counts.argtypes = [vp, vp, vp, vp, vp, vp, i32, i32, vp, WINDOW_FN, vp, vp, vp, vp,
                                                  sz, vp]
            L.hsnct_fhr_stream_counts.restype = i32
            L.hsnct_sync.argtypes = [vp, vp]
            L.hsnct_sync.restype = i32
            L.hsnct_kernel_launches.argtypes = [vp]
            L.hsnct_kernel_launches.restype = ctypes.c_uint64
            L.hsnct_status_string.argtypes = [i32]
            L.hsnct_status_string.restype = ctypes.c_char_p
            L.hsnct_last_error.argtypes = []
            L.hsnct_last_error.restype = ctypes.c_char_p
            L.hsnct_fmd_transform.argtypes = [vp, vp, vp, i32, vp, vp, sz, vp]
            L.hsnct_fmd_transform.restype = i32
            L.hsnct_fmd_materials.argtypes = [vp, vp, vp, i32, vp, vp, sz, vp]
            L.hsnct_fmd_materials.restype = i32
            L.hsnct_fmd_spectra.argtypes = [vp, vp, vp, i32, vp, vp]
            L.hsnct_fmd_spectra.restype = i32
            L.hsnct_debug_trace.argtypes = [vp, vp, sz, ctypes.POINTER(sz), ctypes.POINTER(ctypes.c_int)]
            L.hsnct_debug_trace.restype = i32
            L.hsnct_nmf_red_size.argtypes = [vp]
            L.hsnct_nmf_red_size.restype = sz
            L.hsnct_nmf_begin.argtypes = [vp, vp, i64, vp, vp, sz, vp]
            L.hsnct_nmf_begin.restype = i32
            L.hsnct_nmf_rowpass.argtypes = [vp, vp, i64, vp, vp, i32, vp, sz, vp, vp]
            L.hsnct_nmf_rowpass.restype = i32
            L.hsnct_nmf_dupdate.argtypes = [vp, vp, vp, i32, vp, vp, sz, vp]
            L.hsnct_nmf_dupdate.restype = i32
            L.hsnct_decompose_stats.argtypes = [vp, ctypes.POINTER(i64), vp]
            L.hsnct_decompose_stats.restype = i32
            L.hsnct_debug_plan.argtypes = [vp, ctypes.c_char_p, sz]
            L.hsnct_debug_plan.restype = i32
            L.hsnct_debug_fbp_timing.argtypes = [vp, ctypes.c_int]
            L.hsnct_debug_fbp_timing.restype = i32
            L.hsnct_debug_fbp_times.argtypes = [vp, vp]
            L.hsnct_debug_fbp_times.restype = i32
            L.hsnct_debug_nmf_timing.argtypes = [vp, ctypes.c_int]
            L.hsnct_debug_nmf_timing.restype = i32
            L.hsnct_debug_nmf_times.argtypes = [vp, vp]
            L.hsnct_debug_nmf_times.restype = i32
            L.hsnct_abi_version.argtypes = []
            L.hsnct_abi_version.restype = i32
            _lib = L
    return _lib


def _check(st: int):
    if st != OK:
        L = lib()
        raise HsnctError(st, f"{L.hsnct_status_string(st).decode()}: {L.hsnct_last_error().decode()}")


def _ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream(stream, device):
    s = torch.cuda.current_stream(device) if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


class Hsnct:
    """One handle per geometry (N_v, N_r, N_c, N_k, K) and device."""

    def __init__(self, n_views, n_rows, n_cols, n_bins, n_sub, angles=None, device=0):
        if not torch.cuda.is_available():
            raise HsnctError(E_CUDA, "no CUDA device: the hot path has no CPU fallback")
        self.device = torch.device("cuda", device if isinstance(device, int) else torch.device(device).index or 0)
        self.Nv, self.Nr, self.Nc, self.Nk, self.K = n_views, n_rows, n_cols, n_bins, n_sub
        self.Np = n_views * n_rows * n_cols
        self.Nx = n_rows * n_cols * n_cols
        L = lib()
        self._angles = None
        ap = None
        if angles is not None:
            import numpy as np
            self._angles = np.ascontiguousarray(angles, dtype=np.float64)
            ap = self._angles.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        g = _Geom(n_views, n_rows, n_cols, n_bins, n_sub, ap)
        h = ctypes.c_void_p()
        _check(L.hsnct_create(ctypes.byref(g), self.device.index, ctypes.byref(h)))
        self._h = h
        self._ws = {}

    # -- lifetime -----------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().hsnct_destroy(self._h)
            self._h = None
            self._ws.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def kernel_launches(self) -> int:
        return int(lib().hsnct_kernel_launches(self._h))

    def workspace_bytes(self, op: int) -> int:
        return int(lib().hsnct_workspace_bytes(self._h, op))

    def workspace(self, op: int, nbytes: int | None = None) -> torch.Tensor:
        need = self.workspace_bytes(op) if nbytes is None else nbytes
        ws = self._ws.get(op)
        if ws is None or ws.numel() < need:
            ws = torch.empty(max(need, 256), dtype=torch.uint8, device=self.device)
            self._ws[op] = ws
        return ws

    def release_workspaces(self):
        """Drop the workspaces this handle cached (their device memory returns to torch)."""
        self._ws.clear()

    # -- checks ---------------------------------------------------------------------
    def _dev(self, t, name, shape=None, contiguous=True):
        if not isinstance(t, torch.Tensor) or t.device != self.device or t.dtype != torch.float32:
            raise HsnctError(E_ARG, f"{name} must be a float32 tensor on {self.device}")
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise HsnctError(E_ARG, f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
        if contiguous and not t.is_contiguous():
            raise HsnctError(E_ARG, f"{name} must be contiguous")
        return t

    def _rows(self, t, name, nrows, ncols):
        self._dev(t, name, contiguous=False)
        if t.dim() != 2 or t.shape[0] != nrows or t.shape[1] != ncols or t.stride(1) != 1:
            raise HsnctError(E_ARG, f"{name} must be [{nrows}, {ncols}] with unit column stride")
        return t.stride(0)

    # -- the C ABI calls ------------------------------------------------------------
    def subspace_decompose(self, Y, V, D, n_iter, obj_trace=None, ws=None, stream=None):
        """Eq. 4 by Lee-Seung MU; V, D updated in place (hsnct_subspace_decompose)."""
        ld = self._rows(Y, "Y", self.Np, self.Nk)
        self._dev(V, "V", (self.Np, self.K))
        self._dev(D, "D", (self.K, self.Nk))
        if obj_trace is not None and (obj_trace.dtype != torch.float64 or obj_trace.device != self.device
                                      or obj_trace.numel() < 2 * n_iter or not obj_trace.is_contiguous()):
            raise HsnctError(E_ARG, "obj_trace must be a contiguous float64 device tensor of 2*n_iter")
        ws = self.workspace(OP_DECOMPOSE) if ws is None else ws
        _check(lib().hsnct_subspace_decompose(self._h, _ptr(Y), ld, _ptr(V), _ptr(D), int(n_iter),
                                              _ptr(obj_trace), _ptr(ws), ws.numel() * ws.element_size(),
                                              _stream(stream, self.device)))
        return V, D

    # -- sharded decomposition (NEXT-4): the iteration split at its exchange step -------------
    def nmf_red_size(self) -> int:
        return int(lib().hsnct_nmf_red_size(self._h))

    def nmf_begin(self, Y, D, ws=None, stream=None):
        """Y+ preparation and G = D D^T for a sharded decomposition (hsnct_nmf_begin)."""
        ld = self._rows(Y, "Y", self.Np, self.Nk)
        self._dev(D, "D", (self.K, self.Nk))
        ws = self.workspace(OP_DECOMPOSE) if ws is None else ws
        _check(lib().hsnct_nmf_begin(self._h, _ptr(Y), ld, _ptr(D), _ptr(ws), ws.numel() * ws.element_size(),
                                     _stream(stream, self.device)))

    def nmf_rowpass(self, Y, V, D, it, red, ws=None, stream=None):
        """This rank's row pass of iteration `it`; its sums -> red (hsnct_nmf_rowpass)."""
        ld = self._rows(Y, "Y", self.Np, self.Nk)
        self._dev(V, "V", (self.Np, self.K))
        self._dev(D, "D", (self.K, self.Nk))
        if red.dtype != torch.float64 or red.device != self.device or red.numel() < self.nmf_red_size():
            raise HsnctError(E_ARG, "red must be a float64 device tensor of nmf_red_size() values")
        ws = self.workspace(OP_DECOMPOSE) if ws is None else ws
        _check(lib().hsnct_nmf_rowpass(self._h, _ptr(Y), ld, _ptr(V), _ptr(D), int(it), _ptr(ws),
                                       ws.numel() * ws.element_size(), _ptr(red), _stream(stream, self.device)))

    def nmf_dupdate(self, D, red, it, obj2=None, ws=None, stream=None):
        """D update of iteration `it` from the all-reduced sums (hsnct_nmf_dupdate)."""
        self._dev(D, "D", (self.K, self.Nk))
        ws = self.workspace(OP_DECOMPOSE) if ws is None else ws
        _check(lib().hsnct_nmf_dupdate(self._h, _ptr(D), _ptr(red), int(it), _ptr(obj2), _ptr(ws),
                                       ws.numel() * ws.element_size(), _stream(stream, self.device)))

    def fbp(self, V, X=None, ws=None, stream=None):
        """FBP of the K subspace sinograms -> X [K, N_r, N_c, N_c] (hsnct_fbp)."""
        self._dev(V, "V", (self.Np, self.K))
        if X is None:
            X = torch.empty((self.K, self.Nr, self.Nc, self.Nc), dtype=torch.float32, device=self.device)
        self._dev(X, "X", (self.K, self.Nr, self.Nc, self.Nc))
        ws = self.workspace(OP_FBP) if ws is None else ws
        _check(lib().hsnct_fbp(self._h, _ptr(V), _ptr(X), _ptr(ws), ws.numel() * ws.element_size(),
                               _stream(stream, self.device)))
        return X

    def _counts(self, y, y0, b):
        for t, name, shape in ((y, "y", (self.Np, self.Nk)), (y0, "y0", (self.Nr * self.Nc, self.Nk))):
            if not isinstance(t, torch.Tensor) or t.dtype != torch.uint8 or t.device != self.device \
                    or tuple(t.shape) != shape or not t.is_contiguous():
                raise HsnctError(E_ARG, f"{name} must be a contiguous uint8 tensor {shape} on {self.device}")
        if b is not None:
            self._dev(b, "b", (self.Nv, self.Nk))

    def counts_to_projections(self, y, y0, b=None, Y=None, stream=None):
        """Eq. 2 + Appendix A on uint8 counts (hsnct_counts_to_projections) -> Y [N_p, N_k]."""
        self._counts(y, y0, b)
        if Y is None:
            Y = torch.empty((self.Np, self.Nk), dtype=torch.float32, device=self.device)
        ld = self._rows(Y, "Y", self.Np, self.Nk)
        _check(lib().hsnct_counts_to_projections(self._h, _ptr(y), _ptr(y0), _ptr(b) if b is not None else None,
                                                 _ptr(Y), ld, _stream(stream, self.device)))
        return Y

    def subspace_decompose_counts(self, y, y0, V, D, n_iter, b=None, obj_trace=None, ws=None, stream=None):
        """hsnct_subspace_decompose on Y decoded from uint8 counts (hsnct_subspace_decompose_counts)."""
        self._counts(y, y0, b)
        self._dev(V, "V", (self.Np, self.K))
        self._dev(D, "D", (self.K, self.Nk))
        if obj_trace is not None and (obj_trace.dtype != torch.float64 or obj_trace.device != self.device
                                      or obj_trace.numel() < 2 * n_iter or not obj_trace.is_contiguous()):
            raise HsnctError(E_ARG, "obj_trace must be a contiguous float64 device tensor of 2*n_iter")
        ws = self.workspace(OP_DECOMPOSE_COUNTS) if ws is None else ws
        _check(lib().hsnct_subspace_decompose_counts(self._h, _ptr(y), _ptr(y0), _ptr(b) if b is not None else None,
                                                     _ptr(V), _ptr(D), int(n_iter),
                                                     _ptr(obj_trace) if obj_trace is not None else None, _ptr(ws),
                                                     ws.numel() * ws.element_size(), _stream(stream, self.device)))
        return V, D

    def mbir(self, V, X, n_iter, sigma_v, sigma_x, p=1.2, q=2.0, T=1.0, obj_trace=None, ws=None, stream=None):
        """Eq. 5 MBIR of the K subspace sinograms (hsnct_mbir): X [K, N_r, N_c, N_c] holds x0 and
        is overwritten with the n_iter-th SQS iterate; obj_trace (fp64 [n_iter + 1]) optional."""
        self._dev(V, "V", (self.Np, self.K))
        self._dev(X, "X", (self.K, self.Nr, self.Nc, self.Nc))
        if obj_trace is not None and (obj_trace.dtype != torch.float64 or obj_trace.device != self.device
                                      or obj_trace.numel() < n_iter + 1 or not obj_trace.is_contiguous()):
            raise HsnctError(E_ARG, f"obj_trace must be a contiguous float64 tensor of >= {n_iter + 1} entries")
        prm = MbirParams(float(sigma_v), float(sigma_x), float(p), float(q), float(T))
        ws = self.workspace(OP_MBIR) if ws is None else ws
        _check(lib().hsnct_mbir(self._h, _ptr(V), _ptr(X), int(n_iter), ctypes.byref(prm),
                                _ptr(obj_trace) if obj_trace is not None else None, _ptr(ws),
                                ws.numel() * ws.element_size(), _stream(stream, self.device)))
        return X

    def project(self, X, P=None, ws=None, stream=None):
        """Forward projection A X of Eq. 5 (hsnct_project) -> P [N_p, K] (the layout of V)."""
        self._dev(X, "X", (self.K, self.Nr, self.Nc, self.Nc))
        if P is None:
            P = torch.empty((self.Np, self.K), dtype=torch.float32, device=self.device)
        self._dev(P, "P", (self.Np, self.K))
        ws = self.workspace(OP_PROJECT) if ws is None else ws
        _check(lib().hsnct_project(self._h, _ptr(X), _ptr(P), _ptr(ws), ws.numel() * ws.element_size(),
                                   _stream(stream, self.device)))
        return P

    def synthesize(self, X, D, slice0=0, n_slices=None, bin0=0, n_bins=None, Xh=None, stream=None):
        """x^h window = x^s (D^s)^T (hsnct_synthesize) -> Xh [n_slices*N_c^2, n_bins]."""
        n_slices = self.Nr - slice0 if n_slices is None else n_slices
        n_bins = self.Nk - bin0 if n_bins is None else n_bins
        self._dev(X, "X", (self.K, self.Nr, self.Nc, self.Nc))
        self._dev(D, "D", (self.K, self.Nk))
        if Xh is None:
            Xh = torch.empty((n_slices * self.Nc * self.Nc, n_bins), dtype=torch.float32, device=self.device)
        ld = self._rows(Xh, "Xh", n_slices * self.Nc * self.Nc, n_bins) if Xh.numel() else max(n_bins, 1)
        _check(lib().hsnct_synthesize(self._h, _ptr(X), _ptr(D), slice0, n_slices, bin0, n_bins,
                                      _ptr(Xh), ld, _stream(stream, self.device)))
        return Xh

    def dhr(self, Y, slice0=0, n_slices=None, bin0=0, n_bins=None, Xh=None, ws=None, stream=None):
        """Per-bin FBP baseline (hsnct_dhr) -> Xh [n_slices*N_c^2, n_bins]."""
        n_slices = self.Nr - slice0 if n_slices is None else n_slices
        n_bins = self.Nk - bin0 if n_bins is None else n_bins
        ld_y = self._rows(Y, "Y", self.Np, self.Nk)
        if Xh is None:
            Xh = torch.empty((n_slices * self.Nc * self.Nc, n_bins), dtype=torch.float32, device=self.device)
        ld = self._rows(Xh, "Xh", n_slices * self.Nc * self.Nc, n_bins) if Xh.numel() else max(n_bins, 1)
        if ws is None:
            per = self.workspace_bytes(OP_DHR)  # one slice, all bins
            ws = self.workspace(OP_DHR, per * max(1, min(n_slices, 8)))
        _check(lib().hsnct_dhr(self._h, _ptr(Y), ld_y, slice0, n_slices, bin0, n_bins, _ptr(Xh), ld,
                               _ptr(ws), ws.numel() * ws.element_size(), _stream(stream, self.device)))
        return Xh

    def fhr_host(self, Y, V0, D0, n_iter, Xh=None, V=None, D=None, ws=None, stream=None):
        """Algorithm 1 end to end on HOST tensors (hsnct_fhr_host); blocks until Xh is on the host."""
        for t, name in ((Y, "Y"), (V0, "V0"), (D0, "D0")):
            if t.device.type != "cpu" or t.dtype != torch.float32:
                raise HsnctError(E_ARG, f"{name} must be a float32 host tensor")
        if Y.dim() != 2 or Y.shape != (self.Np, self.Nk) or Y.stride(1) != 1:
            raise HsnctError(E_ARG, "Y must be [N_p, N_k] with unit column stride")
        V0 = V0.contiguous()
        D0 = D0.contiguous()
        if Xh is None:
            Xh = torch.empty((self.Nx, self.Nk), dtype=torch.float32, pin_memory=True)
        if not Xh.is_contiguous() or Xh.shape != (self.Nx, self.Nk):
            raise HsnctError(E_ARG, "Xh must be a contiguous [N_x, N_k] host tensor")
        ws = self.workspace(OP_FHR_HOST) if ws is None else ws
        _check(lib().hsnct_fhr_host(self._h, _ptr(Y), Y.stride(0), _ptr(V0), _ptr(D0), int(n_iter),
                                    _ptr(Xh), _ptr(V), _ptr(D), _ptr(ws), ws.numel() * ws.element_size(),
                                    _stream(stream, self.device)))
        return Xh

    def fhr_stream_window_slices(self, budget_bytes: int = 2 << 30) -> int:
        """Default x^h window (slices) of fhr_stream: the largest that fits budget_bytes."""
        per = self.Nc * self.Nc * self.Nk * 4
        return max(1, min(self.Nr, budget_bytes // per))

    def fhr_stream_ring(self, window_slices: int) -> torch.Tensor:
        """A page-locked host ring of two x^h windows for fhr_stream."""
        return torch.empty((2, window_slices * self.Nc * self.Nc, self.Nk), dtype=torch.float32, pin_memory=True)

    def fhr_stream(self, Y, V0, D0, n_iter, window_slices=None, ring=None, on_window=None, V=None, D=None,
                   ws=None, stream=None):
        """Algorithm 1 end to end on HOST tensors with x^h streamed out in windows
        (hsnct_fhr_stream).  on_window(slice0, n_slices, xh) is called on this thread for every
        window as soon as it is on the host; xh is a [n_slices*N_c*N_c, N_k] view into the ring,
        valid only during the call.  Blocks until the last window has been delivered."""
        if Y.device.type != "cpu" or Y.dtype != torch.float32:
            raise HsnctError(E_ARG, "Y must be a float32 host tensor")
        if Y.dim() != 2 or Y.shape != (self.Np, self.Nk) or Y.stride(1) != 1:
            raise HsnctError(E_ARG, "Y must be [N_p, N_k] with unit column stride")
        return self._fhr_stream(("Y", Y), V0, D0, n_iter, window_slices, ring, on_window, V, D, ws, stream)

    def fhr_stream_counts(self, y, y0, V0, D0, n_iter, b=None, window_slices=None, ring=None, on_window=None,
                          V=None, D=None, ws=None, stream=None):
        """fhr_stream from the detector counts (hsnct_fhr_stream_counts, NEXT-1 end to end): HOST
        uint8 y [N_p, N_k] and y0 [N_r*N_c, N_k], optional fp32 offset b [N_v, N_k]; Eq. 2 is
        decoded on the device.  Results equal fhr_stream on the decoded Y."""
        for t, name, shape in ((y, "y", (self.Np, self.Nk)), (y0, "y0", (self.Nr * self.Nc, self.Nk))):
            if t.device.type != "cpu" or t.dtype != torch.uint8 or tuple(t.shape) != shape or not t.is_contiguous():
                raise HsnctError(E_ARG, f"{name} must be a contiguous uint8 host tensor {shape}")
        if b is not None and (b.device.type != "cpu" or b.dtype != torch.float32 or
                              tuple(b.shape) != (self.Nv, self.Nk) or not b.is_contiguous()):
            raise HsnctError(E_ARG, "b must be a contiguous float32 host tensor [N_v, N_k]")
        return self._fhr_stream(("counts", (y, y0, b)), V0, D0, n_iter, window_slices, ring, on_window, V, D, ws,
                                stream)

    def _fhr_stream(self, src, V0, D0, n_iter, window_slices, ring, on_window, V, D, ws, stream):
        for t, name in ((V0, "V0"), (D0, "D0")):
            if t.device.type != "cpu" or t.dtype != torch.float32:
                raise HsnctError(E_ARG, f"{name} must be a float32 host tensor")
        V0 = V0.contiguous()
        D0 = D0.contiguous()
        wsl = self.fhr_stream_window_slices() if window_slices is None else int(window_slices)
        wsl = max(1, min(wsl, self.Nr))
        if ring is None:
            ring = self.fhr_stream_ring(wsl)
        if not ring.is_contiguous() or ring.numel() < 2 * wsl * self.Nc * self.Nc * self.Nk or ring.device.type != "cpu":
            raise HsnctError(E_ARG, "ring must be a contiguous host tensor of two windows")
        L = lib()
        counts = src[0] == "counts"
        if ws is None:
            nb = (L.hsnct_fhr_stream_counts_bytes if counts else L.hsnct_fhr_stream_bytes)(self._h, wsl)
            ws = torch.empty(nb, dtype=torch.uint8, device=self.device)
        per = self.Nc * self.Nc * self.Nk
        base = ring.data_ptr()
        flat = ring.reshape(-1)
        err = []

        def cb(_user, s0, ns, ptr):
            try:
                if on_window is not None:
                    off = (ptr - base) // 4
                    on_window(s0, ns, flat[off:off + ns * per].view(ns * self.Nc * self.Nc, self.Nk))
            except BaseException as e:  # noqa: BLE001 -- re-raised after the C call returns
                err.append(e)

        fn = WINDOW_FN(cb)
        nbytes = ws.numel() * ws.element_size()
        if counts:
            y, y0, b = src[1]
            _check(L.hsnct_fhr_stream_counts(self._h, _ptr(y), _ptr(y0), _ptr(b), _ptr(V0), _ptr(D0), int(n_iter),
                                             wsl, _ptr(ring), fn, None, _ptr(V), _ptr(D), _ptr(ws), nbytes,
                                             _stream(stream, self.device)))
        else:
            Y = src[1]
            _check(L.hsnct_fhr_stream(self._h, _ptr(Y), Y.stride(0), _ptr(V0), _ptr(D0), int(n_iter), wsl,
                                      _ptr(ring), fn, None, _ptr(V), _ptr(D), _ptr(ws), nbytes,
                                      _stream(stream, self.device)))
        if err:
            raise err[0]
        return ring

    # -- FMD back half (NEXT-2; Algorithm 2) ---------------------------
    def fmd_transform(self, X, labels, n_mat, T=None, ws=None, stream=None):
        """Eq. 7: T [n_mat, K] region means of X [K, N_r, N_c, N_c] (hsnct_fmd_transform)."""
        self._dev(X, "X", (self.K, self.Nr, self.Nc, self.Nc))
        if (not isinstance(labels, torch.Tensor) or labels.dtype != torch.int32 or labels.device != self.device
                or labels.numel() != self.Nx or not labels.is_contiguous()):
            raise HsnctError(E_ARG, f"labels must be a contiguous int32 tensor of {self.Nx} elements on {self.device}")
        if T is None:
            T = torch.empty((n_mat, self.K), dtype=torch.float32, device=self.device)
        self._dev(T, "T", (n_mat, self.K))
        ws = self.workspace(OP_FMD) if ws is None else ws
        _check(lib().hsnct_fmd_transform(self._h, _ptr(X), _ptr(labels), int(n_mat), _ptr(T), _ptr(ws),
                                         ws.numel() * ws.element_size(), _stream(stream, self.device)))
        return T

    def fmd_materials(self, X, T, Xm=None, ws=None, stream=None):
        """Eq. 8: Xm [n_mat, N_r, N_c, N_c], per-voxel NNLS (hsnct_fmd_materials)."""
        n_mat = T.shape[0]
        self._dev(X, "X", (self.K, self.Nr, self.Nc, self.Nc))
        self._dev(T, "T", (n_mat, self.K))
        if Xm is None:
            Xm = torch.empty((n_mat, self.Nr, self.Nc, self.Nc), dtype=torch.float32, device=self.device)
        self._dev(Xm, "Xm", (n_mat, self.Nr, self.Nc, self.Nc))
        ws = self.workspace(OP_FMD) if ws is None else ws
        _check(lib().hsnct_fmd_materials(self._h, _ptr(X), _ptr(T), int(n_mat), _ptr(Xm), _ptr(ws),
                                         ws.numel() * ws.element_size(), _stream(stream, self.device)))
        return Xm

    def fmd_spectra(self, D, T, Dm=None, stream=None):
        """Eq. 9: (D^m)^T = T D, [n_mat, N_k] (hsnct_fmd_spectra)."""
        n_mat = T.shape[0]
        self._dev(D, "D", (self.K, self.Nk))
        self._dev(T, "T", (n_mat, self.K))
        if Dm is None:
            Dm = torch.empty((n_mat, self.Nk), dtype=torch.float32, device=self.device)
        self._dev(Dm, "Dm", (n_mat, self.Nk))
        _check(lib().hsnct_fmd_spectra(self._h, _ptr(D), _ptr(T), int(n_mat), _ptr(Dm), _stream(stream, self.device)))
        return Dm

    def decompose_stats(self, stream=None) -> dict:
        """Statistics of the last subspace_decompose: {"n_clamped": negative Y entries set to 0}."""
        n = ctypes.c_int64(0)
        _check(lib().hsnct_decompose_stats(self._h, ctypes.byref(n), _stream(stream, self.device)))
        return {"n_clamped": int(n.value)}

    def debug_plan(self) -> str:
        """The subspace-extraction plan (row-pass kernel, template, grid) chosen at create."""
        buf = ctypes.create_string_buffer(256)
        _check(lib().hsnct_debug_plan(self._h, buf, 256))
        return buf.value.decode()

    def debug_fbp_timing(self, on: bool):
        """Record CUDA events around the ramp filter and backprojection of later fbp calls."""
        _check(lib().hsnct_debug_fbp_timing(self._h, 1 if on else 0))

    def debug_fbp_times(self):
        """(ramp filter ms, backprojection ms) of the last timed fbp call (waits for it)."""
        ms = (ctypes.c_float * 2)()
        _check(lib().hsnct_debug_fbp_times(self._h, ctypes.cast(ms, ctypes.c_void_p)))
        return float(ms[0]), float(ms[1])

    def debug_nmf_timing(self, on: bool):
        """Record CUDA events around the input preparation and the iterations of later decompose calls."""
        _check(lib().hsnct_debug_nmf_timing(self._h, 1 if on else 0))

    def debug_nmf_times(self):
        """(input preparation ms, iterations ms) of the last timed decompose call (waits for it)."""
        ms = (ctypes.c_float * 2)()
        _check(lib().hsnct_debug_nmf_times(self._h, ctypes.cast(ms, ctypes.c_void_p)))
        return float(ms[0]), float(ms[1])

    def debug_trace(self):
        """%globaltimer stamps (ns) of the last decompose, uint64 [256, n_cta, 16]: per
        iteration (persistent kernel) or per tile of the last iteration (tcgen05 pass, its
        first 256 tiles); None when tracing is off (HSNCT_TRACE=1 at create)."""
        import numpy as np
        L = lib()
        n_out, n_cta = ctypes.c_size_t(0), ctypes.c_int(0)
        _check(L.hsnct_debug_trace(self._h, None, 0, ctypes.byref(n_out), ctypes.byref(n_cta)))
        if n_out.value == 0:
            return None
        buf = np.zeros(n_out.value, dtype=np.uint64)
        _check(L.hsnct_debug_trace(self._h, ctypes.c_void_p(buf.ctypes.data), buf.size, None, None))
        return buf.reshape(-1, n_cta.value, 16)

    def sync(self, stream=None):
        """Wait for the stream; raise the deferred data/numeric status (hsnct_sync)."""
        _check(lib().hsnct_sync(self._h, _stream(stream, self.device)))
