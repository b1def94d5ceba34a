"""B200-native batched tree verification (the server hot path of SpecEdge, arXiv 2505.17052).

The product is libspecedge.so (C ABI in include/specedge.h, CUDA kernels for sm_100a in csrc/);
this package is a thin binding.  It never imports `oracle/`.
"""
from . import _lib  # noqa: F401

__all__ = ["_lib", "api", "build"]
