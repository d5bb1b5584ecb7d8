"""B200-native HE-LRM encrypted embedding lookup (arxiv 2506.18150).

The product is libhelrm.so (C ABI in include/helrm.h, sm_100a kernels in
csrc/); `helrm` is its thin ctypes binding.
"""
__all__ = ["helrm"]
