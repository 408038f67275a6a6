"""paper_2406_06022_b200 -- a B200-native (sm_100a) RGCN mini-batch train step after
GraphStorm (arXiv 2406.06022): libgsb.so (CUDA kernels behind the C ABI in
include/gsb.h) and a thin Python driver.  No CPU fallback: every call fails loudly when
the extension or a CUDA device is missing.
"""
from ._lib import GsbError, lib  # noqa: F401

__all__ = ["GsbError", "lib"]
