"""B200-native CCWSIM hot path (arXiv 2404.00441): wavelet-space CCF pattern
search, top-K selection, conditioning, min-cut stitching and paste on sm_100a.

``ccwsim`` mirrors the reference's ``namespace ccwsim`` API; the numerics run
in libccwgpu.so (CUDA C++ behind the C-ABI in include/ccwgpu.h).
"""
from . import ccwsim  # noqa: F401
from .ccwsim import *  # noqa: F401,F403

__all__ = ["ccwsim"]
