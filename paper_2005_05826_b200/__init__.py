"""stripefrac-b200: B200-native (sm_100a) Striped UniFrac distance-matrix hot path.

``stripefrac`` mirrors the reference C++ API over the C ABI in
``include/stripefrac_cuda.h``; kernels live in ``csrc/``.
"""
from . import stripefrac  # noqa: F401
from ._native import LIB_PATH  # noqa: F401

__all__ = ["stripefrac", "LIB_PATH"]
