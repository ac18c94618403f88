"""Helios (arXiv 2310.00837) mini-batch preparation hot path, B200-native.

The product is libhelios.so (C ABI, include/helios.h, CUDA sm_100a kernels in csrc/); `helios` is
its thin ctypes binding.  Import `paper_2310_00837_b200.helios` explicitly (it fails loudly when the
library has not been built).
"""
__all__ = ["helios", "build"]
