"""B200-native (sm_100a) hot path of fast hyperspectral neutron tomography (arXiv 2410.22500).

The product is libhsnct.so (C ABI, include/hsnct.h) built from csrc/; this
package is its thin binding.  See DESIGN.md.
"""
from .hsnct import Hsnct, HsnctError, lib, LIB_PATH  # noqa: F401

__all__ = ["Hsnct", "HsnctError", "lib", "LIB_PATH"]
