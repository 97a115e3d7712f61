"""B200-native HISA hierarchical indexer (arXiv 2603.28458) behind the reference's proj/core entry points.

The product is the sm_100a library built from csrc/ (C ABI: include/hisa_cuda.h). This package only holds
that library and `capi`, the ctypes binding used by this repo's Python callers; see DESIGN.md.
"""
from . import capi  # noqa: F401

__all__ = ["capi"]
