"""B200-native POAS (predict, optimize, adapt, schedule) co-executed GEMM.

The product is libpoas_b200.so (C++20 planner + runtime, sm_100a CUDA
kernels) behind the C ABI in include/poas_b200.h; this package is its Python
binding. Importing it loads the native library and fails if it is absent.
"""
from . import poas  # noqa: F401
from ._lib import LIB_PATH, PoasError  # noqa: F401

__version__ = "0.1.0"
