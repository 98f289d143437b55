"""B200-native fused MBCI chain E = op(A·B)·D (MCFuser, arXiv 2506.22169).

The product is libmbci.so (C ABI in include/mbci.h, CUDA kernels for sm_100a in csrc/);
``mbci`` is its ctypes binding.  Import ``paper_2506_22169_b200.mbci`` to load the
library (it raises if the library has not been built — there is no CPU fallback).
"""
__all__ = ["mbci", "sharding"]
