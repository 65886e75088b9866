"""CPU-side checks of the C ABI boundary: the library loads, exports every symbol
include/hsnct.h declares, and the host-only error paths behave (no compute)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hsnct.h")


@pytest.fixture(scope="module")
def L():
    from paper_2410_22500_b200 import build as b
    b.build()
    from paper_2410_22500_b200 import hsnct
    return hsnct.lib()


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hsnct_[a-z_]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("hsnct_create", "hsnct_destroy", "hsnct_workspace_bytes", "hsnct_subspace_decompose",
              "hsnct_fbp", "hsnct_synthesize", "hsnct_dhr", "hsnct_fhr_host", "hsnct_sync",
              "hsnct_status_string", "hsnct_last_error", "hsnct_kernel_launches", "hsnct_abi_version",
              "hsnct_fmd_transform", "hsnct_fmd_materials", "hsnct_fmd_spectra", "hsnct_debug_trace",
              "hsnct_debug_fbp_timing", "hsnct_debug_fbp_times", "hsnct_debug_nmf_timing", "hsnct_fhr_stream_counts",
              "hsnct_debug_nmf_times"):
        assert s in syms


def test_library_exports_every_declared_symbol(L):
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = os.popen(f"nm -D --defined-only {L._name}").read()
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), s


def test_library_is_sm100a(L):
    out = os.popen(f"cuobjdump --list-elf {L._name} 2>&1").read()
    assert "sm_100a" in out, out


def test_status_strings_and_version(L):
    assert L.hsnct_abi_version() == 1
    for st in range(6):
        assert L.hsnct_status_string(st)
    assert L.hsnct_status_string(99) == b"unknown status"


def test_null_handle_paths(L):
    vp = ctypes.c_void_p
    assert L.hsnct_workspace_bytes(None, 0) == 0
    assert L.hsnct_kernel_launches(None) == 0
    assert L.hsnct_subspace_decompose(None, None, 0, None, None, 1, None, None, 0, None) == 1
    assert b"handle" in L.hsnct_last_error()
    assert L.hsnct_fbp(None, None, None, None, 0, None) == 1
    assert L.hsnct_synthesize(None, None, None, 0, 0, 0, 0, None, 0, None) == 1
    assert L.hsnct_dhr(None, None, 0, 0, 0, 0, 0, None, 0, None, 0, None) == 1
    assert L.hsnct_fhr_host(None, None, 0, None, None, 0, None, None, None, None, 0, None) == 1
    assert L.hsnct_sync(None, None) == 1
    assert L.hsnct_fmd_transform(None, None, None, 1, None, None, 0, None) == 1
    assert L.hsnct_fmd_materials(None, None, None, 1, None, None, 0, None) == 1
    assert L.hsnct_fmd_spectra(None, None, None, 1, None, None) == 1
    L.hsnct_destroy(None)
    del vp


def test_create_rejects_bad_geometry(L):
    from paper_2410_22500_b200.hsnct import _Geom
    h = ctypes.c_void_p()
    bad = [(1, 1, 16, 8, 2), (8, 0, 16, 8, 2), (8, 1, 1, 8, 2), (8, 1, 2048, 8, 2), (8, 1, 16, 0, 1),
           (8, 1, 16, 8, 0), (8, 1, 16, 8, 17), (8, 1, 16, 4, 5), (8, 1, 16, 8000, 16),
           (8, 1, 1025, 8, 2), (8, 1, 16, 3201, 16)]  # just past the N_c and K*N_kp limits
    for nv, nr, nc, nk, k in bad:
        g = _Geom(nv, nr, nc, nk, k, None)
        assert L.hsnct_create(ctypes.byref(g), 0, ctypes.byref(h)) == 1, (nv, nr, nc, nk, k)
        assert h.value is None
    assert L.hsnct_create(None, 0, ctypes.byref(h)) == 1


def test_create_accepts_the_limits(L):
    """N_c = 1024 and K * round_up(N_k, 4) = 51200 pass the argument checks (include/hsnct.h);
    without a GPU the call then fails on the device query (HSNCT_E_CUDA), not HSNCT_E_ARG."""
    import torch
    from paper_2410_22500_b200.hsnct import _Geom
    for nv, nr, nc, nk, k in [(8, 1, 1024, 8, 2), (8, 1, 16, 3200, 16), (2, 1, 2, 1, 1)]:
        h = ctypes.c_void_p()
        g = _Geom(nv, nr, nc, nk, k, None)
        rc = L.hsnct_create(ctypes.byref(g), 0, ctypes.byref(h))
        if torch.cuda.is_available():
            assert rc == 0, (nv, nr, nc, nk, k, L.hsnct_last_error())
            L.hsnct_destroy(h)
        else:
            assert rc == 4, (nv, nr, nc, nk, k, rc, L.hsnct_last_error())


def test_create_without_gpu_reports_cuda(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2410_22500_b200.hsnct import _Geom
    h = ctypes.c_void_p()
    g = _Geom(8, 1, 16, 8, 2, None)
    assert L.hsnct_create(ctypes.byref(g), 0, ctypes.byref(h)) == 4
    assert b"CUDA" in L.hsnct_last_error() or b"device" in L.hsnct_last_error()


def test_binding_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2410_22500_b200 import Hsnct, HsnctError
    with pytest.raises(HsnctError):
        Hsnct(8, 1, 16, 8, 2)


def test_product_and_oracle_share_nothing():
    """The product never loads the oracle (no CPU fallback) and the oracle never
    includes or links the product."""
    pkg = os.path.join(ROOT, "paper_2410_22500_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cpp", ".cu", ".h", ".cuh")):
                txt = open(os.path.join(dp, f)).read()
                for bad in ("import oracle", "from oracle", "liboracle", "oracle_"):
                    assert bad not in txt, (f, bad)
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".c", ".py", ".h")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            for bad in ('#include "hsnct', '#include "internal', "import paper_2410_22500_b200",
                        "from paper_2410_22500_b200", "libhsnct"):
                assert bad not in txt, (f, bad)
