"""Python mirror of the POAS plan / predict / execute API over the C ABI.

Names and argument meaning follow the reference C++ API (namespace poas,
/root/reference/proj/include/poas/*.hpp); errors raise PoasError whose
`.errc` is the reference's poas::errc name. Every function calls into
libpoas_b200.so -- there is no Python implementation of any of it.
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass
from typing import Sequence

from ._lib import DTYPE_BF16, DTYPE_F16, DTYPE_F32, PoasError, call_str, check, lib, take_string

__all__ = [
    "PoasError", "plan", "plan_standalone", "solve_split", "oracle_grid_search", "build_tile_plan",
    "schedule_roundtrip", "profile_roundtrip", "machine_hash", "fit_linear", "transfer_bytes",
    "solve_simplex", "Unit", "profile_machine", "Executor", "GemmIO", "stream_seed",
    "DTYPE_F32", "DTYPE_F16", "DTYPE_BF16",
]


def _b(s: str) -> bytes:
    return s.encode()


# ------------------------------------------------------------------ planning
def plan(profile: str, m: int, n: int, k: int) -> str:
    """solve_split -> build_tile_plan -> build_schedule -> format_schedule
    (reference proj/tools/poas.cpp:66-83). Returns the schedule JSON text."""
    return call_str(lib.poas_b200_plan, _b(profile), m, n, k)


def plan_policy(profile: str, m: int, n: int, k: int, policy: str = "reference") -> str:
    """plan() under a planner policy: "reference" (byte-identical to the
    reference) or the opt-in "best-subset" B200 extension."""
    return call_str(lib.poas_b200_plan_policy, _b(profile), m, n, k, _b(policy))


def plan_partitions(profile: str, m: int, n: int, k: int, tc_id: str, tc_sms: int, simt_id: str,
                    simt_sms: int, simt_budgets, policy: str = "best-subset") -> dict:
    """The planner's choice of one GPU's SM partition between its tensor and
    CUDA-core units (poas_b200_plan_partitions; B200 extension):
    {"best": i, "candidates": [{"simt_sms", "tc_sms", "makespan", "rows"}]}."""
    arr = (C.c_int * len(simt_budgets))(*[int(x) for x in simt_budgets])
    return json.loads(call_str(lib.poas_b200_plan_partitions, _b(profile), m, n, k, _b(tc_id), int(tc_sms),
                               _b(simt_id), int(simt_sms), arr, len(simt_budgets), _b(policy)))


def splice_unit(profile: str, unit_profile: str, unit_id: str) -> str:
    """`profile` with device `unit_id`'s measured model (slope, intercept,
    bandwidth, ops window) taken from `unit_profile` -- the same unit probed
    again on the SM budget the partition decision gives it
    (poas_b200_profile_splice_unit). Identity, kind, priority and alignment
    stay, so the machine hash is unchanged."""
    return call_str(lib.poas_b200_profile_splice_unit, _b(profile), _b(unit_profile), _b(unit_id))


def refit_profile(profile: str, report: str | dict, alpha: float = 0.5) -> str:
    """Dynamic-scheduling model update (paper §3.4.2; B200 extension): the
    profile re-fitted from one execution report (Executor.execute's dict or
    its JSON text)."""
    if isinstance(report, dict):
        report = json.dumps(report)
    return call_str(lib.poas_b200_refit_profile, _b(profile), _b(report), float(alpha))


def plan_standalone(profile: str, device_id: str, m: int, n: int, k: int) -> str:
    """standalone_schedule (reference proj/src/scheduler.cpp:59-74)."""
    return call_str(lib.poas_b200_plan_standalone, _b(profile), _b(device_id), m, n, k)


def solve_split(profile: str, m: int, n: int, k: int) -> dict:
    """solve_split (reference proj/src/optimizer.cpp:238-325) as a dict."""
    return json.loads(call_str(lib.poas_b200_split, _b(profile), m, n, k))


def oracle_grid_search(profile: str, m: int, n: int, k: int, resolution: int,
                       parallel: bool = True) -> dict:
    """oracle_grid_search(_serial) (reference proj/src/optimizer.cpp:431-439)."""
    return json.loads(call_str(lib.poas_b200_oracle_split, _b(profile), m, n, k, resolution,
                               int(parallel)))


def build_tile_plan(profile: str, m: int, n: int, k: int, rows: Sequence[int]) -> dict:
    """build_tile_plan over evaluate_rows(rows) (reference proj/src/adapter.cpp:171-215)."""
    arr = (C.c_int64 * len(rows))(*rows)
    return json.loads(call_str(lib.poas_b200_tile_plan, _b(profile), m, n, k, arr, len(rows)))


def schedule_roundtrip(text: str) -> str:
    """parse_schedule -> format_schedule (reference proj/src/scheduler.cpp:147-242)."""
    return call_str(lib.poas_b200_schedule_roundtrip, _b(text))


def profile_roundtrip(text: str) -> str:
    """parse_profile -> format_profile (reference proj/src/profiler.cpp:139-209)."""
    return call_str(lib.poas_b200_profile_roundtrip, _b(text))


def machine_hash(profile: str) -> str:
    buf = C.create_string_buffer(17)
    check(lib.poas_b200_machine_hash(_b(profile), buf))
    return buf.value.decode()


def fit_linear(ops: Sequence[int], seconds: Sequence[float]) -> tuple[float, float]:
    """fit_linear (reference proj/src/device_model.cpp:97-131): (slope, intercept)."""
    n = len(ops)
    o = (C.c_uint64 * n)(*ops)
    s = (C.c_double * n)(*seconds)
    slope, icpt = C.c_double(), C.c_double()
    check(lib.poas_b200_fit_linear(o, s, n, C.byref(slope), C.byref(icpt)))
    return slope.value, icpt.value


def transfer_bytes(profile: str, device_id: str, ops: int, m: int, n: int, k: int) -> tuple[int, int]:
    i, o = C.c_uint64(), C.c_uint64()
    check(lib.poas_b200_transfer_bytes(_b(profile), _b(device_id), ops, m, n, k, C.byref(i),
                                       C.byref(o)))
    return i.value, o.value


def solve_simplex(objective, eq_a=(), eq_b=(), ge_a=(), ge_b=()):
    """solve_simplex (reference proj/src/simplex.cpp:86-187): (x, objective, iterations)."""
    nv = len(objective)

    def mat(rows):
        flat = [float(v) for r in rows for v in r]
        return (C.c_double * max(1, len(flat)))(*flat)

    x = (C.c_double * max(1, nv))()
    obj, it = C.c_double(), C.c_long()
    check(lib.poas_b200_simplex(nv, (C.c_double * nv)(*objective), len(eq_a), mat(eq_a),
                                (C.c_double * max(1, len(eq_b)))(*eq_b), len(ge_a), mat(ge_a),
                                (C.c_double * max(1, len(ge_b)))(*ge_b), x, C.byref(obj),
                                C.byref(it)))
    return list(x)[:nv], obj.value, it.value


def stream_seed(master: int, name: str) -> int:
    """Rng::for_stream(master, name) seed (reference proj/include/poas/rng.hpp:43-50)."""
    return lib.poas_b200_stream_seed(master, _b(name))


# ------------------------------------------------------------------- predict
class Unit:
    """One compute unit as a DeviceBackend (reference proj/include/poas/backend.hpp).

    spec: "<id>=<kind>[:key=value]*", e.g. "gpu0.tc=xpu:dev=0:sms=146:dtype=bf16".
    """

    def __init__(self, spec: str):
        self._h = C.c_void_p()
        self._destroy = lib.poas_b200_unit_destroy  # still bound at interpreter exit
        check(lib.poas_b200_unit_create(_b(spec), C.byref(self._h)))

    def time_gemm(self, side: int) -> float:
        s = C.c_double()
        check(lib.poas_b200_time_gemm(self._h, side, C.byref(s)))
        return s.value

    def time_transfer(self, nbytes: int) -> float:
        s = C.c_double()
        check(lib.poas_b200_time_transfer(self._h, nbytes, C.byref(s)))
        return s.value

    def has_transfers(self) -> bool:
        return bool(lib.poas_b200_has_transfers(self._h))

    def close(self):
        if getattr(self, "_h", None):
            self._destroy(self._h)
            self._h = None

    __del__ = close


def profile_machine(units: str, profiling: str = "", bus: bool = True, retries: int = 0) -> str:
    """profile_machine over real units -> "poas-profile v1" text
    (reference proj/src/simulator.cpp:53-74 + proj/src/profiler.cpp:75-135).
    `retries`: re-measure up to that many times when the reference's
    fit_linear rejects the samples (a non-positive slope: host-CPU probes
    of small sides on a busy host); the fit itself is unchanged."""
    for attempt in range(retries + 1):
        try:
            return call_str(lib.poas_b200_profile_machine, _b(units), _b(profiling), int(bus))
        except PoasError as e:
            if e.errc != "degenerate_samples" or attempt == retries:
                raise
    raise AssertionError("unreachable")


GEMM_CB = C.CFUNCTYPE(C.c_double, C.c_void_p, C.c_int64)
TRANSFER_CB = C.CFUNCTYPE(C.c_double, C.c_void_p, C.c_uint64)
KINDS = {"cpu": 0, "gpu": 1, "xpu": 2}


class ProbeBackend(C.Structure):
    """poas_probe_backend (include/poas_b200.h): the C form of the reference
    plugin DeviceBackend (proj/include/poas/backend.hpp:11-24)."""
    _fields_ = [
        ("id", C.c_char_p), ("kind", C.c_int), ("elem_size", C.c_uint32), ("align", C.c_int64),
        ("cache_bytes", C.c_uint64), ("priority", C.c_int), ("probe_min_side", C.c_int64),
        ("probe_max_side", C.c_int64), ("time_gemm", GEMM_CB), ("time_transfer", TRANSFER_CB),
        ("ctx", C.c_void_p),
    ]


def profile_backends(devices, profiling: str = "", bus: bool = True) -> str:
    """profile_machine over caller-supplied backends -> "poas-profile v1".
    `devices`: dicts with id, kind ("cpu"|"gpu"|"xpu"), elem_size, time_gemm
    (side -> seconds) and optionally time_transfer (bytes -> seconds),
    align, cache_bytes, priority (None = ranked), probe_range (min, max).
    A Python exception inside a callback is re-raised after the call."""
    errors = []

    def wrap(fn, cb_type):
        if fn is None:
            return cb_type()

        def cb(_ctx, x):
            try:
                return float(fn(x))
            except BaseException as e:  # noqa: BLE001 -- re-raised below
                errors.append(e)
                return float("nan")
        return cb_type(cb)

    keep = []
    arr = (ProbeBackend * len(devices))()
    for i, d in enumerate(devices):
        g, t = wrap(d["time_gemm"], GEMM_CB), wrap(d.get("time_transfer"), TRANSFER_CB)
        keep += [g, t, d["id"].encode()]
        lo, hi = d.get("probe_range") or (0, 0)
        prio = d.get("priority")
        arr[i] = ProbeBackend(keep[-1], KINDS[d["kind"]], int(d["elem_size"]), int(d.get("align", 0)),
                              int(d.get("cache_bytes", 0)), -1 if prio is None else int(prio),
                              int(lo), int(hi), g, t, None)
    out = C.c_void_p()
    rc = lib.poas_b200_profile_backends(C.cast(arr, C.c_void_p), len(devices), _b(profiling),
                                        int(bus), C.byref(out))
    if errors:
        raise errors[0]
    check(rc)
    return take_string(out)


# ------------------------------------------------------------------- execute
class GemmIO(C.Structure):
    """poas_gemm_io (include/poas_b200.h)."""
    _fields_ = [
        ("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64),
        ("a_host", C.c_void_p), ("lda_host", C.c_int64),
        ("b_host", C.c_void_p), ("ldb_host", C.c_int64),
        ("c_host", C.c_void_p), ("ldc_host", C.c_int64),
        ("a_dev", C.c_void_p), ("lda_dev", C.c_int64),
        ("b_dev", C.c_void_p), ("ldb_dev", C.c_int64),
        ("a16_dev", C.c_void_p), ("lda16_dev", C.c_int64),
        ("b16_dev", C.c_void_p), ("ldb16_dev", C.c_int64),
        ("c_dev", C.c_void_p), ("ldc_dev", C.c_int64),
        ("resident", C.c_int),
        ("b_panels", C.c_int), ("b_ready", C.POINTER(C.c_void_p)),
        ("a16_host", C.c_void_p), ("lda16_host", C.c_int64),
        ("b16_host", C.c_void_p), ("ldb16_host", C.c_int64),
        ("b_flags", C.c_void_p), ("b_epoch", C.c_int),
        ("comm", C.c_void_p), ("b_transport", C.c_int),
    ]


class Executor:
    """The real replacement of simulate() (reference proj/src/simulator.cpp:104-209)."""

    def __init__(self, units: str):
        self._h = C.c_void_p()
        self._destroy = lib.poas_b200_executor_destroy  # still bound at interpreter exit
        check(lib.poas_b200_executor_create(_b(units), C.byref(self._h)))

    @property
    def machine_hash(self) -> str:
        buf = C.create_string_buffer(17)
        check(lib.poas_b200_executor_hash(self._h, buf))
        return buf.value.decode()

    def execute(self, schedule: str, io: GemmIO, repeats: int = 1) -> dict:
        out = C.c_void_p()
        check(lib.poas_b200_execute(self._h, _b(schedule), C.byref(io), repeats, C.byref(out)))
        from ._lib import take_string
        return json.loads(take_string(out))

    def run_dynamic(self, profile: str, m: int, n: int, k: int, io: GemmIO, iterations: int,
                    policy: str = "reference", alpha: float = 0.5,
                    replan_threshold_pct: float = 2.0, repeats: int = 1) -> dict:
        """Dynamic scheduling loop (poas_b200_run_dynamic): plan, execute
        `repeats` times back to back, re-fit, re-plan when |makespan error| >
        threshold; per-iteration log, the final profile and schedule."""
        out = C.c_void_p()
        check(lib.poas_b200_run_dynamic(self._h, _b(profile), m, n, k, _b(policy), C.byref(io),
                                        iterations, repeats, float(alpha),
                                        float(replan_threshold_pct), C.byref(out)))
        from ._lib import take_string
        return json.loads(take_string(out))

    def close(self):
        if getattr(self, "_h", None):
            self._destroy(self._h)
            self._h = None

    __del__ = close


# ----------------------------------------------------------------- multi-GPU
TRANSPORTS = {"ce": 0, "nccl": 1}


class Comm:
    """poas_comm_t: the job's ranks joined through shared memory, B moved
    by copy engines over CUDA IPC (or NCCL). `device` -1: host-only."""

    def __init__(self, name: str, rank: int, world: int, device: int = -1):
        self._h = C.c_void_p()
        self._destroy = lib.poas_b200_comm_destroy
        check(lib.poas_b200_comm_create(_b(name), rank, world, device, C.byref(self._h)))
        self.rank, self.world, self.device = rank, world, device

    @property
    def handle(self) -> int:
        return self._h.value

    def barrier(self):
        check(lib.poas_b200_comm_barrier(self._h))

    def allgather(self, text: str) -> list[str]:
        return json.loads(call_str(lib.poas_b200_comm_allgather, self._h, _b(text)))

    def max(self, value: float) -> float:
        out = C.c_double()
        check(lib.poas_b200_comm_max(self._h, float(value), C.byref(out)))
        return out.value

    def init_nccl(self):
        """Rank 0 makes an NCCL id, every rank joins (collective)."""
        hexid = ""
        if self.rank == 0:
            buf = (C.c_ubyte * 512)()
            n = C.c_size_t()
            check(lib.poas_b200_nccl_unique_id(buf, 512, C.byref(n)))
            hexid = bytes(buf[:n.value]).hex()
        hexid = self.allgather(hexid)[0]
        raw = bytes.fromhex(hexid)
        check(lib.poas_b200_comm_init_nccl(self._h, (C.c_ubyte * len(raw)).from_buffer_copy(raw), len(raw)))

    def register_b(self, b16: int, b32: int | None, k: int, n: int, panels: int):
        check(lib.poas_b200_comm_register_b(self._h, b16, b32, k, n, panels))

    def time_broadcast(self, nbytes: int, transport: str = "ce", repetitions: int = 3) -> float:
        out = C.c_double()
        check(lib.poas_b200_comm_time_broadcast(self._h, _b(transport), nbytes, repetitions, C.byref(out)))
        return out.value

    def close(self):
        if getattr(self, "_h", None):
            self._destroy(self._h)
            self._h = None

    __del__ = close


def plan_sharded(gpu_profiles: Sequence[str], link_bandwidth: Sequence[float], m: int, n: int, k: int,
                 policy: str = "reference") -> dict:
    """Two-level plan (poas/sharded.hpp): rows per GPU from the level-1
    plan, then each GPU's own plan of its rows."""
    g = len(gpu_profiles)
    profs = (C.c_char_p * g)(*[_b(p) for p in gpu_profiles])
    bw = (C.c_double * g)(*[float(x) for x in link_bandwidth])
    return json.loads(call_str(lib.poas_b200_plan_sharded, profs, bw, g, m, n, k, _b(policy)))


# --------------------------------------------------------------- raw kernels
def tc_gemm(dtype: int, m, n, k, a, lda, b, ldb, c, ldc, accumulate=False, num_ctas=0, stream=None):
    check(lib.poas_b200_tc_gemm(dtype, m, n, k, a, lda, b, ldb, c, ldc, int(accumulate), num_ctas,
                                stream))


def tc_gemm_panels(dtype: int, m, n, k, a, lda, b, ldb, c, ldc, panels, flags=None, epoch=0,
                   accumulate=False, num_ctas=0, stream=None):
    """One launch over panel-major B; panel p gated on flags[p] >= epoch."""
    check(lib.poas_b200_tc_gemm_panels(dtype, m, n, k, a, lda, b, ldb, c, ldc, int(accumulate),
                                       num_ctas, panels, flags, epoch, stream))


def signal_flag(flag_ptr: int, value: int, stream=None):
    """*flag = value in `stream` order (cuStreamWriteValue32)."""
    check(lib.poas_b200_signal_flag(flag_ptr, value, stream))


def tc_kernel_name(m: int, n: int, k: int) -> str:
    """The tensor-core kernel tc_gemm launches for this shape."""
    return lib.poas_b200_tc_kernel_name(m, n, k).decode()


def tc_scheduler_name(m: int, n: int, k: int) -> str:
    """The tile scheduler tc_gemm uses for this shape ("dynamic" or "wave")."""
    return lib.poas_b200_tc_scheduler_name(m, n, k).decode()


def simt_gemm(m, n, k, a, lda, b, ldb, c, ldc, accumulate=False, num_ctas=0, exclusive=False,
              stream=None):
    check(lib.poas_b200_simt_gemm(m, n, k, a, lda, b, ldb, c, ldc, int(accumulate), num_ctas,
                                  int(exclusive), stream))


def host_gemm(m, n, k, a, lda, b, ldb, c, ldc, accumulate=False, threads=0):
    check(lib.poas_b200_host_gemm(m, n, k, a, lda, b, ldb, c, ldc, int(accumulate), threads))


def fill_uniform(dtype, dst, ld, rows, cols, row0, col0, total_cols, seed, stream=None):
    check(lib.poas_b200_fill_uniform(dtype, dst, ld, rows, cols, row0, col0, total_cols, seed, stream))


def fill_uniform_host(dst, ld, rows, cols, row0, col0, total_cols, seed):
    check(lib.poas_b200_fill_uniform_host(dst, ld, rows, cols, row0, col0, total_cols, seed))


def convert_f32(dtype, src, ld_src, dst, ld_dst, rows, cols, stream=None):
    check(lib.poas_b200_convert_f32(dtype, src, ld_src, dst, ld_dst, rows, cols, stream))


def sm_count() -> int:
    return lib.poas_b200_sm_count()
