"""B200-native FireQ W4A8-FP linear layer (arXiv 2505.20839).

The product is libfireq.so (C ABI in include/fireq.h, CUDA kernels for sm_100a in
csrc/); `fireq` is its ctypes binding and `sharding` the column-parallel host
logic.  Import of this package does not load the library; fireq.load() does.
"""
__all__ = ["fireq", "sharding"]
