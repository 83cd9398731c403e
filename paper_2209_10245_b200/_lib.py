"""ctypes binding of libpoas_b200.so (the C ABI declared in include/poas_b200.h).

The shared library is the product: every call below goes into native code.
If the library is missing the import fails loudly -- there is no fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libpoas_b200.so"

i64 = C.c_int64
u64 = C.c_uint64
vp = C.c_void_p
dp = C.POINTER(C.c_double)
cp = C.c_char_p
pcp = C.POINTER(C.c_char_p)

# name -> (restype, argtypes)
SIGNATURES: dict[str, tuple] = {
    "poas_b200_last_error": (cp, []),
    "poas_b200_free": (None, [vp]),
    "poas_b200_version": (cp, []),
    "poas_b200_plan": (C.c_int, [cp, i64, i64, i64, C.POINTER(vp)]),
    "poas_b200_plan_standalone": (C.c_int, [cp, cp, i64, i64, i64, C.POINTER(vp)]),
    "poas_b200_plan_policy": (C.c_int, [cp, i64, i64, i64, cp, C.POINTER(vp)]),
    "poas_b200_profile_splice_unit": (C.c_int, [cp, cp, cp, C.POINTER(vp)]),
    "poas_b200_plan_partitions": (C.c_int, [cp, i64, i64, i64, cp, C.c_int, cp, C.c_int,
                                            C.POINTER(C.c_int), C.c_int, cp, C.POINTER(vp)]),
    "poas_b200_split": (C.c_int, [cp, i64, i64, i64, C.POINTER(vp)]),
    "poas_b200_oracle_split": (C.c_int, [cp, i64, i64, i64, i64, C.c_int, C.POINTER(vp)]),
    "poas_b200_tile_plan": (C.c_int, [cp, i64, i64, i64, C.POINTER(i64), C.c_size_t, C.POINTER(vp)]),
    "poas_b200_schedule_roundtrip": (C.c_int, [cp, C.POINTER(vp)]),
    "poas_b200_profile_roundtrip": (C.c_int, [cp, C.POINTER(vp)]),
    "poas_b200_machine_hash": (C.c_int, [cp, C.c_char_p]),
    "poas_b200_fit_linear": (C.c_int, [C.POINTER(u64), dp, C.c_size_t, dp, dp]),
    "poas_b200_transfer_bytes": (C.c_int, [cp, cp, u64, i64, i64, i64, C.POINTER(u64), C.POINTER(u64)]),
    "poas_b200_simplex": (C.c_int, [C.c_int, dp, C.c_int, dp, dp, C.c_int, dp, dp, dp, dp,
                                    C.POINTER(C.c_long)]),
    "poas_b200_unit_create": (C.c_int, [cp, C.POINTER(vp)]),
    "poas_b200_unit_destroy": (None, [vp]),
    "poas_b200_time_gemm": (C.c_int, [vp, i64, dp]),
    "poas_b200_time_transfer": (C.c_int, [vp, u64, dp]),
    "poas_b200_has_transfers": (C.c_int, [vp]),
    "poas_b200_profile_machine": (C.c_int, [cp, cp, C.c_int, C.POINTER(vp)]),
    "poas_b200_profile_backends": (C.c_int, [vp, C.c_size_t, cp, C.c_int, C.POINTER(vp)]),
    "poas_b200_executor_create": (C.c_int, [cp, C.POINTER(vp)]),
    "poas_b200_executor_destroy": (None, [vp]),
    "poas_b200_execute": (C.c_int, [vp, cp, vp, C.c_int, C.POINTER(vp)]),
    "poas_b200_executor_hash": (C.c_int, [vp, C.c_char_p]),
    "poas_b200_tc_kernel_name": (cp, [i64, i64, i64]),
    "poas_b200_tc_scheduler_name": (cp, [i64, i64, i64]),
    "poas_b200_refit_profile": (C.c_int, [cp, cp, C.c_double, C.POINTER(vp)]),
    "poas_b200_run_dynamic": (C.c_int, [vp, cp, i64, i64, i64, cp, vp, C.c_int, C.c_int, C.c_double,
                                        C.c_double, C.POINTER(vp)]),
    "poas_b200_comm_create": (C.c_int, [cp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "poas_b200_comm_destroy": (None, [vp]),
    "poas_b200_comm_barrier": (C.c_int, [vp]),
    "poas_b200_comm_allgather": (C.c_int, [vp, cp, C.POINTER(vp)]),
    "poas_b200_comm_max": (C.c_int, [vp, C.c_double, dp]),
    "poas_b200_nccl_unique_id": (C.c_int, [vp, C.c_size_t, C.POINTER(C.c_size_t)]),
    "poas_b200_comm_init_nccl": (C.c_int, [vp, vp, C.c_size_t]),
    "poas_b200_comm_register_b": (C.c_int, [vp, vp, vp, i64, i64, C.c_int]),
    "poas_b200_comm_time_broadcast": (C.c_int, [vp, cp, u64, C.c_int, dp]),
    "poas_b200_plan_sharded": (C.c_int, [C.POINTER(cp), dp, C.c_int, i64, i64, i64, cp, C.POINTER(vp)]),
    "poas_b200_tc_gemm": (C.c_int, [C.c_int, i64, i64, i64, vp, i64, vp, i64, vp, i64, C.c_int,
                                    C.c_int, vp]),
    "poas_b200_tc_gemm_panels": (C.c_int, [C.c_int, i64, i64, i64, vp, i64, vp, i64, vp, i64, C.c_int,
                                           C.c_int, C.c_int, vp, C.c_int, vp]),
    "poas_b200_signal_flag": (C.c_int, [vp, C.c_int, vp]),
    "poas_b200_wait_flag": (C.c_int, [vp, C.c_int, vp]),
    "poas_b200_simt_gemm": (C.c_int, [i64, i64, i64, vp, i64, vp, i64, vp, i64, C.c_int, C.c_int,
                                      C.c_int, vp]),
    "poas_b200_host_gemm": (C.c_int, [i64, i64, i64, vp, i64, vp, i64, vp, i64, C.c_int, C.c_int]),
    "poas_b200_fill_uniform": (C.c_int, [C.c_int, vp, i64, i64, i64, i64, i64, i64, u64, vp]),
    "poas_b200_fill_uniform_host": (C.c_int, [vp, i64, i64, i64, i64, i64, i64, u64]),
    "poas_b200_convert_f32": (C.c_int, [C.c_int, vp, i64, vp, i64, i64, i64, vp]),
    "poas_b200_sm_count": (C.c_int, []),
    "poas_b200_stream_seed": (u64, [u64, cp]),
}

ERROR_NAMES = {
    0: "ok", 1: "invalid_argument", 2: "degenerate_samples", 3: "non_positive_time",
    4: "backend_failure", 5: "parse_failure", 6: "not_row_aligned", 7: "unalignable_k",
    8: "no_feasible_tiling", 9: "too_many_devices", 10: "missing_device",
    11: "numerical_failure", 12: "hash_mismatch", 13: "io_failure", 100: "cuda", 101: "internal",
}

DTYPE_F32, DTYPE_F16, DTYPE_BF16 = 0, 1, 2


class PoasError(RuntimeError):
    """A non-zero return from the C ABI; `.code` is the ABI code, `.errc`
    the reference's poas::errc name (proj/include/poas/error.hpp:8-21)."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[{ERROR_NAMES.get(code, code)}] {message}")
        self.code = code
        self.errc = ERROR_NAMES.get(code, str(code))
        self.message = message


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2209_10245_b200.build` "
            "(there is no non-native fallback)")
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)  # AttributeError if the export is missing
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> None:
    if rc != 0:
        msg = lib.poas_b200_last_error()
        raise PoasError(rc, msg.decode() if msg else "")


def take_string(p: C.c_void_p) -> str:
    """Copies a library-allocated char* and frees it."""
    try:
        return C.string_at(p).decode()
    finally:
        lib.poas_b200_free(p)


def call_str(fn, *args) -> str:
    out = vp()
    check(fn(*args, C.byref(out)))
    return take_string(out)
