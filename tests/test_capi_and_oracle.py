"""CPU-side checks: the C-ABI library loads and exports every declared
symbol; error codes mirror poas::errc; the oracle matches its golden
vectors; the host CPU unit and a CPU-only executor run are exact."""
import json
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT


def declared_symbols():
    text = (ROOT / "include" / "poas_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(poas_b200_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2209_10245_b200 import _lib

    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    names = declared_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python binding covers all of them
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)


def test_error_codes_mirror_reference_errc():
    hdr = (ROOT / "include" / "poas_b200.h").read_text()
    order = ["INVALID_ARGUMENT", "DEGENERATE_SAMPLES", "NON_POSITIVE_TIME", "BACKEND_FAILURE",
             "PARSE_FAILURE", "NOT_ROW_ALIGNED", "UNALIGNABLE_K", "NO_FEASIBLE_TILING",
             "TOO_MANY_DEVICES", "MISSING_DEVICE", "NUMERICAL_FAILURE", "HASH_MISMATCH", "IO_FAILURE"]
    for i, name in enumerate(order, start=1):
        assert re.search(rf"POAS_E_{name} = {i},", hdr), name
    # reference enum order (proj/include/poas/error.hpp:8-21)
    ref = (ROOT / "paper_2209_10245_b200" / "csrc" / "include" / "poas" / "error.hpp").read_text()
    body = ref.split("enum class errc {")[1].split("};")[0]
    assert [w.strip().rstrip(",").upper() for w in body.split() if w.strip()] == order


def test_errors_carry_codes(poas):
    from paper_2209_10245_b200 import PoasError

    with pytest.raises(PoasError) as e:
        poas.plan("not a profile", 1, 1, 1)
    assert e.value.errc == "parse_failure" and "line 1" in e.value.message
    prof = (GOLDEN / "profiles" / "mach2_exact.profile").read_text()
    with pytest.raises(PoasError) as e:
        poas.plan(prof, 0, 10, 10)
    assert e.value.errc == "invalid_argument"
    with pytest.raises(PoasError) as e:
        poas.plan_standalone(prof, "nope", 10, 10, 10)
    assert e.value.errc == "missing_device"
    with pytest.raises(PoasError) as e:
        poas.oracle_grid_search(prof.replace("device xpu0", "device xpu0") + prof.split("device cpu0")[1]
                                .replace("cpu0", "cpu9").join(["\ndevice cpu9", ""]).replace(
                                    "priority 2", "priority 7"), 100, 100, 100, 10)
    assert e.value.errc in ("too_many_devices", "parse_failure", "invalid_argument")
    with pytest.raises(PoasError) as e:
        poas.Unit("x=tpu")
    assert e.value.errc == "invalid_argument"


def test_oracle_rng_golden():
    """Rng::for_stream(20261017, "A").next_u64() = 14442304120711173584 and
    next_unit() = 0.78291887516857028 (from the
    reference library)."""
    import oracle

    g = json.loads((GOLDEN / "rng.json").read_text())
    assert g["for_stream_20261017_A"][0] == 14442304120711173584
    assert g["for_stream_20261017_A"][1] == 0.78291887516857028
    seed = oracle.stream_seed(20261017, "A")
    lib = oracle.oracle_lib()
    assert lib.oracle_draw(seed, 0) == g["for_stream_20261017_A"][0]
    assert lib.oracle_draw(seed, 9) == g["for_stream_20261017_A_draw9"][0]
    assert lib.oracle_draw(oracle.stream_seed(20261017, "B"), 0) == g["for_stream_20261017_B"][0]
    x = oracle.fill_uniform(1, 1, seed)
    assert x[0, 0] == np.float32(2 * 0.78291887516857028 - 1)


def test_product_generator_matches_oracle(poas):
    import oracle

    seed = poas.stream_seed(20261017, "B")
    assert seed == oracle.stream_seed(20261017, "B")
    host = np.empty((33, 65), dtype=np.float32)
    poas.fill_uniform_host(host.ctypes.data, 65, 33, 65, 4, 9, 1000, seed)
    assert np.array_equal(host, oracle.fill_uniform(33, 65, seed, 4, 9, 1000))


def test_oracle_gemm_and_rounding_vs_numpy():
    import oracle

    A, B = oracle.fill_uniform(37, 53, 1), oracle.fill_uniform(53, 29, 2)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert np.allclose(oracle.gemm_rows_f64(A, B, 0), ref, rtol=0, atol=1e-12)
    # bf16 RNE against torch's conversion
    import torch

    x = np.random.default_rng(1).standard_normal(10000).astype(np.float32) * 7
    assert np.array_equal(oracle.round_to(x, 2), torch.from_numpy(x).bfloat16().float().numpy())
    assert np.array_equal(oracle.round_to(x, 1), torch.from_numpy(x).half().float().numpy())
    tiny = np.array([1e-6, -3e-7, 6.1e-5, 65519.0, 65520.0, 1e-8], dtype=np.float32)
    assert np.array_equal(oracle.round_to(tiny, 1), torch.from_numpy(tiny).half().float().numpy())


def test_oracle_tile_execution_matches_full_product():
    import oracle

    A, B = oracle.fill_uniform(64, 96, 3), oracle.fill_uniform(96, 40, 4)
    out = oracle.exec_tiles_f32(A, B, [30, 34] * 3, 32)  # 3 strips x 2 parts
    assert oracle.rel_frobenius(out, oracle.gemm_rows_f64(A, B, 0)) <= 1e-6


@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 33, 5), (100, 200, 300), (257, 129, 64), (6, 32, 1000)])
def test_host_gemm_unit_vs_oracle(poas, shape):
    import oracle

    m, n, k = shape
    A, B = oracle.fill_uniform(m, k, 7), oracle.fill_uniform(k, n, 8)
    C = np.full((m, n), np.nan, dtype=np.float32)
    poas.host_gemm(m, n, k, A.ctypes.data, k, B.ctypes.data, n, C.ctypes.data, n, threads=4)
    assert oracle.rel_frobenius(C, oracle.gemm_rows_f64(A, B, 0)) <= 2e-5
    C0 = oracle.fill_uniform(m, n, 9)
    C2 = C0.copy()
    poas.host_gemm(m, n, k, A.ctypes.data, k, B.ctypes.data, n, C2.ctypes.data, n, accumulate=True)
    assert oracle.rel_frobenius(C2, oracle.gemm_rows_f64(A, B, 0) + C0) <= 2e-5


def test_cpu_only_executor_run(poas, ref):
    """The executor's host path (no GPU needed): profile a CPU unit, plan the
    config C1 shape (scaled), execute, check C and the report."""
    import oracle

    units = "cpu0=cpu:threads=4"
    profile = poas.profile_machine(units, "probes=4,repetitions=3,cpu_min_side=192,cpu_max_side=448", retries=3)
    m, n, k = 300, 256, 128
    sched = poas.plan(profile, m, n, k)
    assert sched == ref.plan(profile, m, n, k)
    A, B = oracle.fill_uniform(m, k, 1), oracle.fill_uniform(k, n, 2)
    C = np.full((m, n), np.nan, dtype=np.float32)
    io = poas.GemmIO(m=m, n=n, k=k, a_host=A.ctypes.data, lda_host=k, b_host=B.ctypes.data,
                     ldb_host=n, c_host=C.ctypes.data, ldc_host=n, resident=1)
    ex = poas.Executor(units)
    rep = ex.execute(sched, io, 2)
    assert oracle.rel_frobenius(C, oracle.gemm_rows_f64(A, B, 0)) <= 2e-5
    d = rep["devices"][0]
    assert d["rows"] == m and d["compute"]["measured"] > 0 and d["copy_in"]["measured"] == 0
    assert rep["measured_makespan"] == pytest.approx(d["finish"]["measured"])
    # machine tokens (shared link, lending, overlapped / pipelined copies)
    # leave a host-only run and the machine identity unchanged
    ex2 = poas.Executor(units + ";bus=1;lend=0;overlap=1;pipeline=1")
    assert ex2.machine_hash == ex.machine_hash
    C[:] = np.nan
    ex2.execute(sched, io, 1)
    assert oracle.rel_frobenius(C, oracle.gemm_rows_f64(A, B, 0)) <= 2e-5


def test_unit_spec_parsing(poas):
    from paper_2209_10245_b200 import PoasError

    for bad in ["", "x", "=cpu", "a=cpu:threads", "a=cpu:threads=x", "a=xpu:dtype=fp8",
                "a=gpu:probe=9-3", "a=gpu:link=nvlink", "a=gpu:bogus=1"]:
        with pytest.raises(PoasError):
            poas.Executor(bad)
    with pytest.raises(PoasError) as e:
        poas.Executor("a=cpu;a=cpu")
    assert e.value.errc == "invalid_argument"
