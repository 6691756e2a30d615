"""B200-native LucidRaster: sort-middle exact order-independent transparency.

The product is libveil.so (C++ host + sm_100a CUDA kernels) behind the
reference's C ABI (include/veil.h) plus additive extensions
(include/veil_cuda.h). This package holds its sources (csrc/), the Makefile
and a thin ctypes binding (veil.py) used by tests and bench.py.
"""
from .abi import default_params, SceneArrays  # noqa: F401
