"""TEST INFRASTRUCTURE -- the CPU checkers. Importable only from tests/,
bench.py (cpu_baseline and --impl reference) and __graft_entry__.smoke().

  ref       the reference planner itself (oracle/_ref/libpoasref.so, compiled
            from /root/reference/proj/src by oracle/Makefile) behind the same
            JSON/text formats as the product's C ABI -- plan parity is checked
            byte for byte against it;
  gemm_*    the fp64 C restatement (oracle/gemm_oracle.c) -- C-value parity
            is UNPINNED by the reference, which has no GEMM.
"""
from __future__ import annotations

import ctypes as C
import json
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libpoasref.so"
ORACLE_SO = HERE / "liboracle.so"

i64, u64, vp, cp = C.c_int64, C.c_uint64, C.c_void_p, C.c_char_p
dp = C.POINTER(C.c_double)


def build(with_ref: bool = True) -> None:
    """make the C oracle (and, when /root/reference exists, the reference lib)."""
    targets = ["oracle"]
    if with_ref and Path("/root/reference/proj/src").is_dir():
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_ref = None
_orc = None


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        lib = C.CDLL(str(REF_SO))
        sig = {
            "ref_last_error": (cp, []), "ref_free": (None, [vp]),
            "ref_plan": (C.c_int, [cp, i64, i64, i64, C.POINTER(vp)]),
            "ref_plan_standalone": (C.c_int, [cp, cp, i64, i64, i64, C.POINTER(vp)]),
            "ref_split": (C.c_int, [cp, i64, i64, i64, C.POINTER(vp)]),
            "ref_oracle_split": (C.c_int, [cp, i64, i64, i64, i64, C.c_int, C.POINTER(vp)]),
            "ref_tile_plan": (C.c_int, [cp, i64, i64, i64, C.POINTER(i64), C.c_size_t, C.POINTER(vp)]),
            "ref_schedule_roundtrip": (C.c_int, [cp, C.POINTER(vp)]),
            "ref_profile_roundtrip": (C.c_int, [cp, C.POINTER(vp)]),
            "ref_machine_hash": (C.c_int, [cp, cp]),
            "ref_fit_linear": (C.c_int, [C.POINTER(u64), dp, C.c_size_t, dp, dp]),
            "ref_transfer_bytes": (C.c_int, [cp, cp, u64, i64, i64, i64, C.POINTER(u64), C.POINTER(u64)]),
            "ref_simplex": (C.c_int, [C.c_int, dp, C.c_int, dp, dp, C.c_int, dp, dp, dp, dp,
                                      C.POINTER(C.c_long)]),
            "ref_profile_synthetic": (C.c_int, [cp, u64, C.POINTER(vp)]),
            "ref_exact_profile": (C.c_int, [cp, C.POINTER(vp)]),
            "ref_probe_trace": (C.c_int, [cp, u64, C.POINTER(vp)]),
            "ref_evaluate_report": (C.c_int, [cp, cp, C.c_int, u64, C.POINTER(vp)]),
            "ref_machine_config_roundtrip": (C.c_int, [cp, C.POINTER(vp)]),
            "ref_rng_draw": (u64, [u64, cp, C.c_int, dp]),
            "ref_time_plan": (C.c_int, [cp, i64, i64, i64, C.c_int, dp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype, f.argtypes = res, args
        _ref = lib
    return _ref


def oracle_lib() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            build(with_ref=False)
        lib = C.CDLL(str(ORACLE_SO))
        sig = {
            "oracle_stream_seed": (u64, [u64, cp]),
            "oracle_draw": (u64, [u64, u64]),
            "oracle_fill_uniform": (None, [vp, i64, i64, i64, i64, i64, i64, u64]),
            "oracle_round": (None, [vp, i64, C.c_int]),
            "oracle_gemm_rows_f64": (None, [i64, i64, i64, vp, i64, vp, i64, vp, i64, C.c_int]),
            "oracle_gemm_rows_f64_strips": (None, [i64, i64, i64, vp, i64, vp, i64, vp, i64]),
            "oracle_rel_frobenius": (C.c_double, [i64, i64, vp, i64, vp, i64]),
            "oracle_exec_tiles_f32": (None, [i64, i64, vp, i64, vp, i64, vp, i64, C.POINTER(i64), i64,
                                             i64, i64]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype, f.argtypes = res, args
        _orc = lib
    return _orc


# --------------------------------------------------------------- reference
def _rcall(fn, *args) -> str:
    lib = ref_lib()
    out = vp()
    rc = fn(*args, C.byref(out))
    if rc != 0:
        raise OracleError(rc, lib.ref_last_error().decode())
    try:
        return C.string_at(out).decode()
    finally:
        lib.ref_free(out)


def ref_check(rc: int) -> None:
    if rc != 0:
        raise OracleError(rc, ref_lib().ref_last_error().decode())


class ref:
    """The reference planner, same signatures as paper_2209_10245_b200.poas."""

    @staticmethod
    def plan(profile, m, n, k):
        return _rcall(ref_lib().ref_plan, profile.encode(), m, n, k)

    @staticmethod
    def plan_standalone(profile, dev, m, n, k):
        return _rcall(ref_lib().ref_plan_standalone, profile.encode(), dev.encode(), m, n, k)

    @staticmethod
    def solve_split(profile, m, n, k):
        return json.loads(_rcall(ref_lib().ref_split, profile.encode(), m, n, k))

    @staticmethod
    def oracle_grid_search(profile, m, n, k, resolution, parallel=True):
        return json.loads(_rcall(ref_lib().ref_oracle_split, profile.encode(), m, n, k, resolution,
                                 int(parallel)))

    @staticmethod
    def build_tile_plan(profile, m, n, k, rows):
        arr = (C.c_int64 * len(rows))(*rows)
        return json.loads(_rcall(ref_lib().ref_tile_plan, profile.encode(), m, n, k, arr, len(rows)))

    @staticmethod
    def schedule_roundtrip(text):
        return _rcall(ref_lib().ref_schedule_roundtrip, text.encode())

    @staticmethod
    def profile_roundtrip(text):
        return _rcall(ref_lib().ref_profile_roundtrip, text.encode())

    @staticmethod
    def machine_hash(profile):
        buf = C.create_string_buffer(17)
        ref_check(ref_lib().ref_machine_hash(profile.encode(), buf))
        return buf.value.decode()

    @staticmethod
    def fit_linear(ops, secs):
        n = len(ops)
        s, c = C.c_double(), C.c_double()
        ref_check(ref_lib().ref_fit_linear((C.c_uint64 * n)(*ops), (C.c_double * n)(*secs), n,
                                           C.byref(s), C.byref(c)))
        return s.value, c.value

    @staticmethod
    def transfer_bytes(profile, dev, ops, m, n, k):
        i, o = C.c_uint64(), C.c_uint64()
        ref_check(ref_lib().ref_transfer_bytes(profile.encode(), dev.encode(), ops, m, n, k,
                                               C.byref(i), C.byref(o)))
        return i.value, o.value

    @staticmethod
    def solve_simplex(objective, eq_a=(), eq_b=(), ge_a=(), ge_b=()):
        nv = len(objective)

        def mat(rows):
            flat = [float(v) for r in rows for v in r]
            return (C.c_double * max(1, len(flat)))(*flat)

        x = (C.c_double * max(1, nv))()
        obj, it = C.c_double(), C.c_long()
        ref_check(ref_lib().ref_simplex(nv, (C.c_double * nv)(*objective), len(eq_a), mat(eq_a),
                                        (C.c_double * max(1, len(eq_b)))(*eq_b), len(ge_a),
                                        mat(ge_a), (C.c_double * max(1, len(ge_b)))(*ge_b), x,
                                        C.byref(obj), C.byref(it)))
        return list(x)[:nv], obj.value, it.value

    @staticmethod
    def profile_synthetic(machine_cfg, seed):
        return _rcall(ref_lib().ref_profile_synthetic, machine_cfg.encode(), seed)

    @staticmethod
    def probe_trace(machine_cfg, seed):
        """Every synthetic-backend measurement the reference profile_machine
        takes, in call order (oracle/ref_shim.cpp ref_probe_trace)."""
        return json.loads(_rcall(ref_lib().ref_probe_trace, machine_cfg.encode(), seed))

    @staticmethod
    def evaluate_report(machine_cfg, inputs, repeats=2, seed=1):
        """The reference evaluate report (format_report_json) for
        `inputs` = [(name, m, n, k), ...] on a synthetic machine."""
        spec = ";".join(f"{nm}:{m}x{n}x{k}" for nm, m, n, k in inputs)
        return json.loads(_rcall(ref_lib().ref_evaluate_report, machine_cfg.encode(), spec.encode(),
                                 repeats, seed))

    @staticmethod
    def exact_profile(machine_cfg):
        return _rcall(ref_lib().ref_exact_profile, machine_cfg.encode())

    @staticmethod
    def machine_config_roundtrip(text):
        return _rcall(ref_lib().ref_machine_config_roundtrip, text.encode())

    @staticmethod
    def rng_draw(master, name, index=0):
        u = C.c_double()
        v = ref_lib().ref_rng_draw(master, name.encode(), index, C.byref(u))
        return v, u.value

    @staticmethod
    def time_plan(profile, m, n, k, reps):
        s = C.c_double()
        ref_check(ref_lib().ref_time_plan(profile.encode(), m, n, k, reps, C.byref(s)))
        return s.value


# ---------------------------------------------------------------- GEMM oracle
def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def stream_seed(master: int, name: str) -> int:
    return oracle_lib().oracle_stream_seed(master, name.encode())


def fill_uniform(rows: int, cols: int, seed: int, row0: int = 0, col0: int = 0,
                 total_cols: int | None = None) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float32)
    oracle_lib().oracle_fill_uniform(_p(out), cols, rows, cols, row0, col0,
                                     cols if total_cols is None else total_cols, seed)
    return out


def round_to(x: np.ndarray, mode: int) -> np.ndarray:
    """mode 0 fp32 (no-op), 1 fp16, 2 bf16 (RNE)."""
    y = np.ascontiguousarray(x, dtype=np.float32).copy()
    oracle_lib().oracle_round(_p(y), y.size, mode)
    return y


def gemm_rows_f64(A: np.ndarray, B: np.ndarray, mode: int) -> np.ndarray:
    """C = round(A) . round(B) with double accumulation (mode as round_to)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    rows, k = A.shape
    k2, n = B.shape
    assert k == k2
    C_ = np.empty((rows, n), dtype=np.float64)
    oracle_lib().oracle_gemm_rows_f64(rows, n, k, _p(A), k, _p(B), n, _p(C_), n, mode)
    return C_


def sampled_rows(m: int, count: int = 64, seed: int = 5) -> np.ndarray:
    """Row indices for a full-size check: the first and last row, the
    boundary rows of 128/256-row tiles (UMMA M, the CTA-pair tile) spread
    over M, and random rows -- sorted, unique, `count` of them (or m)."""
    rng = np.random.default_rng(seed)
    picks = {0, m - 1}
    for t in np.linspace(0, max(0, m // 256 - 1), num=12, dtype=np.int64):
        for off in (0, 127, 128, 255):
            r = int(t) * 256 + off
            if r < m:
                picks.add(r)
    while len(picks) < min(count, m):
        picks.add(int(rng.integers(0, m)))
    return np.array(sorted(picks)[:count] if len(picks) > count else sorted(picks), dtype=np.int64)


def full_size_rows_f64(rows: np.ndarray, n: int, k: int, seed_a: int, seed_b: int, mode: int) -> np.ndarray:
    """Expected C rows of the BASELINE workload at full size: A's sampled
    rows and all of B regenerated from the counter-based stream
    (proj/include/poas/rng.hpp:17-25), rounded to the unit's operand
    precision (`mode`), fp64 accumulation -- one pass over B."""
    A = np.empty((len(rows), k), dtype=np.float32)
    for i, r in enumerate(rows):
        A[i] = fill_uniform(1, k, seed_a, int(r), 0, k)[0]
    B = fill_uniform(k, n, seed_b)
    if mode:
        oracle_lib().oracle_round(_p(A), A.size, mode)
        oracle_lib().oracle_round(_p(B), B.size, mode)
    out = np.empty((len(rows), n), dtype=np.float64)
    oracle_lib().oracle_gemm_rows_f64_strips(len(rows), n, k, _p(A), k, _p(B), n, _p(out), n)
    return out


def rel_frobenius(C32: np.ndarray, R: np.ndarray) -> float:
    C32 = np.ascontiguousarray(C32, dtype=np.float32)
    R = np.ascontiguousarray(R, dtype=np.float64)
    rows, n = C32.shape
    return oracle_lib().oracle_rel_frobenius(rows, n, _p(C32), n, _p(R), n)


def exec_tiles_f32(A: np.ndarray, B: np.ndarray, tile_m: list[int], k_prime: int) -> np.ndarray:
    """CPU execution of one unit's reference tile list (split-K), fp32."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    B = np.ascontiguousarray(B, dtype=np.float32)
    rows, k = A.shape
    n = B.shape[1]
    out = np.empty((rows, n), dtype=np.float32)
    tm = (C.c_int64 * len(tile_m))(*tile_m)
    oracle_lib().oracle_exec_tiles_f32(n, k, _p(A), k, _p(B), n, _p(out), n, tm, len(tile_m),
                                       k_prime, rows)
    return out


def expected_c(schedule: dict, A: np.ndarray, B: np.ndarray, unit_modes: dict[str, int]) -> np.ndarray:
    """The plan semantics: rows contiguous in schedule order, each unit's rows
    computed from its own operand precision, fp64 accumulation."""
    m = A.shape[0]
    out = np.empty((m, B.shape[1]), dtype=np.float64)
    r0 = 0
    for d in schedule["devices"]:
        r = d["rows"]
        if r:
            out[r0:r0 + r] = gemm_rows_f64(A[r0:r0 + r], B, unit_modes.get(d["id"], 0))
        r0 += r
    assert r0 == m
    return out
