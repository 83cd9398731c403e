"""B200-native POAS (predict, optimize, adapt, schedule) co-executed GEMM.

The product is libpoas_b200.so (C++20 planner + runtime, sm_100a CUDA
kernels) behind the C ABI in include/poas_b200.h; `paper_2209_10245_b200.poas`
is its Python binding. Importing the binding loads the native library and
fails loudly if it is absent or stale -- there is no fallback. The package
itself stays import-light so `python -m paper_2209_10245_b200.build` can
(re)build the library first.
"""

__version__ = "0.1.0"


def __getattr__(name):
    if name in ("PoasError", "LIB_PATH"):
        from . import _lib

        return getattr(_lib, name)
    raise AttributeError(name)
