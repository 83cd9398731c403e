"""GPU end-to-end: predict (real units) -> plan (== reference planner) ->
execute through the C ABI -> C checked against the fp64 oracle under the
plan semantics (rows contiguous in schedule order, each unit's own operand
precision). Covers resident (HBM) and host (PCIe copy) runs, a CPU unit in
the co-execution (config C2), error paths and the prediction report shape.
"""
import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 2e-5
SEED = 20261017
PROF = "probes=4,repetitions=2,bandwidth_payload=8388608"


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def operands(torch, poas, m, n, k):
    import oracle

    sa, sb = poas.stream_seed(SEED, "A"), poas.stream_seed(SEED, "B")
    A, B = oracle.fill_uniform(m, k, sa), oracle.fill_uniform(k, n, sb)
    ld16a, ld16b = (k + 7) // 8 * 8, (n + 7) // 8 * 8
    d = {
        "A": A, "B": B,
        "A32": torch.from_numpy(A).cuda(), "B32": torch.from_numpy(B).cuda(),
        "A16": torch.zeros(m, ld16a, device="cuda", dtype=torch.bfloat16),
        "B16": torch.zeros(k, ld16b, device="cuda", dtype=torch.bfloat16),
        "C": torch.full((m, n), float("nan"), device="cuda"),
        "hA": torch.from_numpy(A).pin_memory(), "hB": torch.from_numpy(B).pin_memory(),
        "hC": torch.full((m, n), float("nan")).pin_memory(),
    }
    d["A16"][:, :k] = d["A32"].bfloat16()
    d["B16"][:, :n] = d["B32"].bfloat16()
    d["io_res"] = poas.GemmIO(m=m, n=n, k=k, a_dev=d["A32"].data_ptr(), lda_dev=k,
                              b_dev=d["B32"].data_ptr(), ldb_dev=n, a16_dev=d["A16"].data_ptr(),
                              lda16_dev=ld16a, b16_dev=d["B16"].data_ptr(), ldb16_dev=ld16b,
                              c_dev=d["C"].data_ptr(), ldc_dev=n, a_host=d["hA"].data_ptr(),
                              lda_host=k, b_host=d["hB"].data_ptr(), ldb_host=n,
                              c_host=d["hC"].data_ptr(), ldc_host=n, resident=1)
    d["io_host"] = poas.GemmIO(m=m, n=n, k=k, a_host=d["hA"].data_ptr(), lda_host=k,
                               b_host=d["hB"].data_ptr(), ldb_host=n, c_host=d["hC"].data_ptr(),
                               ldc_host=n, resident=0)
    return d


def result_c(torch, sched, d, resident):
    """Gather C: GPU units wrote c_dev (resident) or c_host; cpu units c_host."""
    out = d["hC"].numpy().copy() if not resident else d["C"].cpu().numpy()
    if resident:
        host = d["hC"].numpy()
        r0 = 0
        for dev in sched["devices"]:
            if dev["id"].startswith("cpu"):
                out[r0:r0 + dev["rows"]] = host[r0:r0 + dev["rows"]]
            r0 += dev["rows"]
    return out


UNITS = ("gpu0.tc=xpu:dev=0:sms=16:dtype=bf16:elem=2:link=hbm:probe=512-2048;"
         "gpu0.simt=gpu:dev=0:sms=8:exclusive=1:elem=4:link=hbm:probe=256-1024")


def test_profile_plan_execute_resident(torch_cuda, poas, ref):
    import oracle

    torch = torch_cuda
    m, n, k = 3000, 1536, 1024
    profile = poas.profile_machine(UNITS, PROF, True)
    assert poas.profile_roundtrip(profile) == profile == ref.profile_roundtrip(profile)
    sched_text = poas.plan(profile, m, n, k)
    assert sched_text == ref.plan(profile, m, n, k)
    sched = json.loads(sched_text)
    ex = poas.Executor(UNITS)
    assert ex.machine_hash == sched["machine_hash"] == poas.machine_hash(profile)
    d = operands(torch, poas, m, n, k)
    rep = ex.execute(sched_text, d["io_res"], 2)
    torch.cuda.synchronize()
    got = result_c(torch, sched, d, True)
    exp = oracle.expected_c(sched, d["A"], d["B"], {"gpu0.tc": 2, "gpu0.simt": 0})
    assert oracle.rel_frobenius(got, exp) <= TOL
    # the reference simulate-report shape (proj/tools/poas.cpp:85-114)
    assert set(rep) >= {"machine_hash", "dims", "seed", "repeats", "predicted_makespan",
                        "measured_makespan", "makespan_error_pct", "devices", "rmse"}
    for dv in rep["devices"]:
        assert set(dv) >= {"id", "rows", "copy_in", "compute", "copy_out", "copy", "finish"}
    assert rep["repeats"] == 2 and rep["measured_makespan"] > 0


def test_execute_host_buffers_over_pcie(torch_cuda, poas):
    import oracle

    torch = torch_cuda
    units = UNITS.replace("elem=2:link=hbm", "elem=4:link=pcie").replace("elem=4:link=hbm", "elem=4:link=pcie")
    m, n, k = 2500, 1024, 768
    profile = poas.profile_machine(units, PROF, True)
    # force both units busy with a hand-made split so both copy paths run
    sched_text = poas.plan(profile, m, n, k)
    sched = json.loads(sched_text)
    d = operands(torch, poas, m, n, k)
    ex = poas.Executor(units)
    rep = ex.execute(sched_text, d["io_host"], 1)
    got = d["hC"].numpy()
    exp = oracle.expected_c(sched, d["A"], d["B"], {"gpu0.tc": 2, "gpu0.simt": 0})
    assert oracle.rel_frobenius(got, exp) <= TOL
    busy = [x for x in rep["devices"] if x["rows"] > 0]
    assert all(x["copy_in"]["measured"] > 0 and x["copy_out"]["measured"] > 0 for x in busy)


def test_every_split_is_exact(torch_cuda, poas):
    """Row-offset convention for arbitrary splits (including 1-row and idle
    units): schedules built from evaluate_rows-style row vectors."""
    import oracle

    torch = torch_cuda
    m, n, k = 777, 640, 512
    profile = poas.profile_machine(UNITS, PROF, True)
    base = json.loads(poas.plan(profile, m, n, k))
    d = operands(torch, poas, m, n, k)
    ex = poas.Executor(UNITS)
    for rows_tc in (0, 8, 384, 769, 776):
        sched = json.loads(json.dumps(base))
        for dv in sched["devices"]:
            dv["rows"] = rows_tc if dv["id"] == "gpu0.tc" else m - rows_tc
        d["C"].fill_(float("nan"))
        ex.execute(json.dumps(sched), d["io_res"], 1)
        torch.cuda.synchronize()
        exp = oracle.expected_c(sched, d["A"], d["B"], {"gpu0.tc": 2, "gpu0.simt": 0})
        assert oracle.rel_frobenius(d["C"].cpu().numpy(), exp) <= TOL, rows_tc


def test_cpu_unit_coexecution_config_c2(torch_cuda, poas, ref):
    """Config C2 shape (scaled): host CPU + CUDA cores + fp16 tensor cores."""
    import oracle

    torch = torch_cuda
    units = ("cpu0=cpu:threads=4;gpu0.simt=gpu:dev=0:sms=2:exclusive=1:elem=4:link=hbm:probe=128-512;"
             "gpu0.tc=xpu:dev=0:sms=4:dtype=f16:elem=2:link=hbm:probe=256-1024")
    m, n, k = 1024, 512, 512
    profile = poas.profile_machine(units, "probes=4,repetitions=2,cpu_min_side=128,cpu_max_side=320,"
                                          "bandwidth_payload=4194304", True)
    sched = json.loads(poas.plan(profile, m, n, k))
    assert json.dumps(sched) == json.dumps(json.loads(ref.plan(profile, m, n, k)))
    # give every unit rows so all three paths execute
    rows = {"cpu0": 16, "gpu0.simt": 40, "gpu0.tc": m - 56}
    for dv in sched["devices"]:
        dv["rows"] = rows[dv["id"]]
    d = operands(torch, poas, m, n, k)
    # fp16 bits in the 16-bit operand buffers (the tensor unit is dtype=f16)
    d["A16"][:, :k] = d["A32"].half().view(torch.bfloat16)
    d["B16"][:, :n] = d["B32"].half().view(torch.bfloat16)
    ex = poas.Executor(units)
    ex.execute(json.dumps(sched), d["io_res"], 1)
    torch.cuda.synchronize()
    got = result_c(torch, sched, d, True)
    exp = oracle.expected_c(sched, d["A"], d["B"], {"gpu0.tc": 1, "gpu0.simt": 0, "cpu0": 0})
    assert oracle.rel_frobenius(got, exp) <= TOL


def test_b_panels_with_ready_events(torch_cuda, poas):
    """Panel-major B arriving panel by panel (the N > 1 broadcast overlap):
    each unit waits on its panel's event; C must be exact regardless."""
    import ctypes

    import oracle

    torch = torch_cuda
    m, n, k, P = 1536, 2048, 512, 4
    np_ = n // P
    profile = poas.profile_machine(UNITS, PROF, True)
    sched = json.loads(poas.plan(profile, m, n, k))
    for dv in sched["devices"]:  # both units busy
        dv["rows"] = 1024 if dv["id"] == "gpu0.tc" else m - 1024
    sched_text = json.dumps(sched)
    d = operands(torch, poas, m, n, k)
    src32, src16 = d["B32"], d["B16"][:, :n]
    B32p = torch.zeros(P, k, np_, device="cuda")
    B16p = torch.zeros(P, k, np_, device="cuda", dtype=torch.bfloat16)
    side = torch.cuda.Stream()
    events = [torch.cuda.Event() for _ in range(P)]
    torch.cuda.synchronize()
    with torch.cuda.stream(side):  # "broadcast": panels land one by one
        for p in range(P):
            torch.cuda._sleep(2_000_000)
            B32p[p].copy_(src32[:, p * np_:(p + 1) * np_])
            B16p[p].copy_(src16[:, p * np_:(p + 1) * np_])
            events[p].record(side)
    handles = (ctypes.c_void_p * P)(*[e.cuda_event for e in events])
    io = poas.GemmIO(m=m, n=n, k=k, a_dev=d["A32"].data_ptr(), lda_dev=k, b_dev=B32p.data_ptr(),
                     ldb_dev=np_, a16_dev=d["A16"].data_ptr(), lda16_dev=d["A16"].shape[1],
                     b16_dev=B16p.data_ptr(), ldb16_dev=np_, c_dev=d["C"].data_ptr(), ldc_dev=n,
                     resident=1, b_panels=P, b_ready=ctypes.cast(handles, ctypes.POINTER(ctypes.c_void_p)))
    ex = poas.Executor(UNITS)
    ex.execute(sched_text, io, 1)
    torch.cuda.synchronize()
    exp = oracle.expected_c(sched, d["A"], d["B"], {"gpu0.tc": 2, "gpu0.simt": 0})
    assert oracle.rel_frobenius(d["C"].cpu().numpy(), exp) <= TOL


def test_execute_error_paths(torch_cuda, poas):
    from paper_2209_10245_b200 import PoasError

    torch = torch_cuda
    profile = poas.profile_machine(UNITS, PROF, True)
    sched = poas.plan(profile, 256, 256, 256)
    d = operands(torch, poas, 256, 256, 256)
    other = poas.Executor(UNITS.replace("gpu0.simt", "gpu0.cuda"))
    with pytest.raises(PoasError) as e:
        other.execute(sched, d["io_res"], 1)
    assert e.value.errc == "hash_mismatch"
    ex = poas.Executor(UNITS)
    with pytest.raises(PoasError) as e:
        ex.execute(sched.replace('"version": 1', '"version": 3'), d["io_res"], 1)
    assert e.value.errc == "parse_failure"
    bad = poas.GemmIO(m=256, n=256, k=256, resident=1)
    with pytest.raises(PoasError) as e:
        ex.execute(sched, bad, 1)
    assert e.value.errc == "invalid_argument"
    with pytest.raises(PoasError):
        ex.execute(sched, d["io_res"], 0)


def test_unit_backend_plugin(torch_cuda, poas):
    u = poas.Unit("gpu0.tc=xpu:dev=0:sms=8:dtype=bf16:elem=2:link=pcie")
    assert u.has_transfers()
    t1, t2 = u.time_gemm(512), u.time_gemm(1000)  # 1000: padded TMA pitch path
    assert 0 < t1 < t2
    assert u.time_transfer(1 << 22) > 0
    c = poas.Unit("cpu0=cpu:threads=2")
    assert not c.has_transfers()
    assert c.time_gemm(64) > 0


def test_dynamic_rescheduling_on_gpu_units(torch_cuda, poas):
    """Dynamic scheduling (paper §3.4.2) on real units: the tensor unit's
    profile is planted 3x too optimistic; the first (static) run misses the
    prediction by ~2/3, the re-fitted plans converge and C stays exact."""
    import oracle

    torch = torch_cuda
    m, n, k = 6000, 3072, 2048  # ~0.7 ms on the test units: kernel time dominates launch latency
    profile = poas.profile_machine(UNITS, PROF, True)
    lines, cur = [], None
    for line in profile.splitlines():
        parts = line.split()
        if len(parts) == 2 and parts[0] == "device":
            cur = parts[1]
        if cur == "gpu0.tc" and len(parts) == 2 and parts[0] in ("slope", "intercept"):
            line = f"{parts[0]} {float(parts[1]) / 4.0!r}"
        lines.append(line)
    planted = "\n".join(lines) + "\n"
    d = operands(torch, poas, m, n, k)
    ex = poas.Executor(UNITS + ";lend=0")
    out = ex.run_dynamic(planted, m, n, k, d["io_res"], iterations=5, alpha=1.0,
                         replan_threshold_pct=2.0)
    torch.cuda.synchronize()
    its = out["iterations"]
    assert its[0]["makespan_error_pct"] > 30.0, its[0]
    assert out["replans"] >= 1
    # converges from ~2/3 off to the unmodelled remainder (launch and
    # cross-stream latency of a sub-millisecond co-executed step)
    best = min(abs(i["makespan_error_pct"]) for i in its[1:])
    assert best < 20.0 and best < 0.5 * its[0]["makespan_error_pct"], its
    assert out["schedule"]["machine_hash"] == ex.machine_hash
    # C holds the last executed plan (rows in schedule order)
    sched = {"devices": [{"id": i, "rows": r} for i, r in its[-1]["rows"].items()]}
    got = result_c(torch, sched, d, True)
    exp = oracle.expected_c(sched, d["A"], d["B"], {"gpu0.tc": 2, "gpu0.simt": 0})
    assert oracle.rel_frobenius(got, exp) <= TOL


def test_sm_lending_idle_units(torch_cuda, poas):
    """A schedule leaving the CUDA-core unit idle: the tensor unit borrows
    its SMs (default) or keeps its own budget ("lend=0"); same identity,
    same exact C."""
    import oracle

    torch = torch_cuda
    m, n, k = 1024, 768, 512
    profile = poas.profile_machine(UNITS, PROF, True)
    sched_text = poas.plan_standalone(profile, "gpu0.tc", m, n, k)
    sched = json.loads(sched_text)
    assert {d["id"]: d["rows"] for d in sched["devices"]}["gpu0.simt"] == 0
    d = operands(torch, poas, m, n, k)
    exp = oracle.expected_c(sched, d["A"], d["B"], {"gpu0.tc": 2, "gpu0.simt": 0})
    for units in (UNITS, UNITS + ";lend=0"):
        ex = poas.Executor(units)
        assert ex.machine_hash == sched["machine_hash"]
        d["C"].fill_(float("nan"))
        ex.execute(sched_text, d["io_res"], 1)
        torch.cuda.synchronize()
        assert oracle.rel_frobenius(result_c(torch, sched, d, True), exp) <= TOL


def test_execute_host_bf16_operands_elem2(torch_cuda, poas):
    """A tensor unit with a 2-byte link copies 16-bit host operands
    (a16_host/b16_host) -- half the PCIe bytes, no conversion pass -- and
    needs no fp32 host A/B when it is the only busy unit."""
    import oracle

    torch = torch_cuda
    units = "gpu0.tc=xpu:dev=0:sms=16:dtype=bf16:elem=2:link=pcie:probe=512-2048"
    m, n, k = 1500, 1000, 516  # k % 8 != 0: staging pads A rows to 8 elements
    profile = poas.profile_machine(units, PROF, True)
    sched_text = poas.plan(profile, m, n, k)
    sched = json.loads(sched_text)
    d = operands(torch, poas, m, n, k)
    hA16 = d["A16"][:, :k].cpu().contiguous().pin_memory()
    hB16 = d["B16"][:, :n].cpu().contiguous().pin_memory()
    hC = torch.full((m, n), float("nan")).pin_memory()
    io = poas.GemmIO(m=m, n=n, k=k, c_host=hC.data_ptr(), ldc_host=n, resident=0,
                     a16_host=hA16.data_ptr(), lda16_host=k, b16_host=hB16.data_ptr(), ldb16_host=n)
    ex = poas.Executor(units)
    rep = ex.execute(sched_text, io, 2)
    exp = oracle.expected_c(sched, d["A"], d["B"], {"gpu0.tc": 2})
    assert oracle.rel_frobenius(hC.numpy(), exp) <= TOL
    tc = [x for x in rep["devices"] if x["id"] == "gpu0.tc"][0]
    assert tc["copy_in"]["measured"] > 0 and tc["copy_out"]["measured"] > 0
    # without 16-bit host operands the unit needs fp32 host A/B
    from paper_2209_10245_b200 import PoasError

    bad = poas.GemmIO(m=m, n=n, k=k, c_host=hC.data_ptr(), ldc_host=n, resident=0)
    with pytest.raises(PoasError):
        ex.execute(sched_text, bad, 1)


def _set_models(profile, slope):
    """Every unit gets the same compute model (a hand-made machine for the
    planner: compute-bound and symmetric, so it splits the rows)."""
    lines = []
    for line in profile.splitlines():
        parts = line.split()
        if len(parts) == 2 and parts[0] == "slope":
            line = f"slope {slope!r}"
        elif len(parts) == 2 and parts[0] == "intercept":
            line = "intercept 0"
        lines.append(line)
    return "\n".join(lines) + "\n"


def test_overlapped_host_execution(torch_cuda, poas):
    """Overlapped copies (executor "overlap=1" + planner policy "overlap"):
    both link units pipeline their row parts -- B and the A parts
    host->device, per-part GEMMs, per-part C device->host on separate
    streams. C is exact for every unit (fp32 host A/B, the tensor unit
    converting on the GPU); the measured phases overlap as planned."""
    import oracle

    torch = torch_cuda
    units = UNITS.replace("elem=2:link=hbm", "elem=4:link=pcie").replace("elem=4:link=hbm", "elem=4:link=pcie")
    m, n, k = 3000, 2048, 1024
    profile = poas.profile_machine(units, PROF, True)
    # a machine on which both units keep rows, so both paths run
    planted = _set_models(profile, 2e-13)
    sched_text = poas.plan_policy(planted, m, n, k, "overlap")
    sched = json.loads(sched_text)
    rows = {d["id"]: d["rows"] for d in sched["devices"]}
    assert rows["gpu0.tc"] > 0 and rows["gpu0.simt"] > 0, rows
    assert all(len(x["tiles"]) > 1 for x in sched["devices"]), sched["devices"]
    d = operands(torch, poas, m, n, k)
    ex = poas.Executor(units + ";overlap=1")
    rep = ex.execute(sched_text, d["io_host"], 3)
    exp = oracle.expected_c(sched, d["A"], d["B"], {"gpu0.tc": 2, "gpu0.simt": 0})
    assert oracle.rel_frobenius(d["hC"].numpy(), exp) <= TOL
    for x in rep["devices"]:
        if x["rows"] > 0:
            assert x["copy_in"]["measured"] > 0 and x["copy_out"]["measured"] > 0
    # the same schedule through a synchronous executor gives the same C
    d["hC"].fill_(float("nan"))
    poas.Executor(units).execute(sched_text, d["io_host"], 1)
    assert oracle.rel_frobenius(d["hC"].numpy(), exp) <= TOL


def test_overlapped_parts_and_bf16_link(torch_cuda, poas):
    """Tensor unit alone with 16-bit host operands, overlapped: every row
    part's C lands (ragged last part, k % 8 != 0), the device->host stream
    starts before the host->device stream ends, and the prediction of the
    pipelined timeline is in the measured range."""
    import oracle

    torch = torch_cuda
    units = "gpu0.tc=xpu:dev=0:sms=16:dtype=bf16:elem=2:link=pcie:probe=512-2048"
    m, n, k = 4000, 4096, 1028
    profile = poas.profile_machine(units, PROF, True)
    sched_text = poas.plan_policy(profile, m, n, k, "overlap")
    sched = json.loads(sched_text)
    tiles = sched["devices"][0]["tiles"]
    panels = [t["n"] for t in tiles[:next(i for i in range(1, len(tiles) + 1)
                                          if sum(x["n"] for x in tiles[:i]) >= n)]]
    assert len(tiles) > 1 and sum(t["m"] for t in tiles) == m * len(panels)
    d = operands(torch, poas, m, n, k)
    hA16 = d["A16"][:, :k].cpu().contiguous().pin_memory()
    hB16 = d["B16"][:, :n].cpu().contiguous().pin_memory()
    hC = torch.full((m, n), float("nan")).pin_memory()
    io = poas.GemmIO(m=m, n=n, k=k, c_host=hC.data_ptr(), ldc_host=n, resident=0,
                     a16_host=hA16.data_ptr(), lda16_host=k, b16_host=hB16.data_ptr(), ldb16_host=n)
    ex = poas.Executor(units + ";overlap=1")
    rep = ex.execute(sched_text, io, 3)
    exp = oracle.expected_c(sched, d["A"], d["B"], {"gpu0.tc": 2})
    assert oracle.rel_frobenius(hC.numpy(), exp) <= TOL
    tc = rep["devices"][0]
    # phase spans are measured on the unit's own three streams
    assert tc["copy_in"]["measured"] > 0 and tc["copy_out"]["measured"] > 0
    assert rep["measured_makespan"] < (tc["copy_in"]["measured"] + tc["compute"]["measured"]
                                       + tc["copy_out"]["measured"])
    assert abs(rep["makespan_error_pct"]) < 60.0, rep["makespan_error_pct"]


def test_b_panels_with_flags_one_launch(torch_cuda, poas):
    """Resident run with panel-major B and device readiness flags: the
    tensor unit consumes all panels in one launch gated per panel; flags
    delivered late on another stream; C exact."""
    import oracle

    torch = torch_cuda
    units = "gpu0.tc=xpu:dev=0:sms=16:dtype=bf16:elem=2:link=hbm:probe=512-2048"
    m, n, k, P = 1500, 1024, 384, 4
    profile = poas.profile_machine(units, PROF, True)
    sched_text = poas.plan(profile, m, n, k)
    sched = json.loads(sched_text)
    d = operands(torch, poas, m, n, k)
    np_ = n // P
    good = torch.stack([d["B16"][:, p * np_:(p + 1) * np_] for p in range(P)]).contiguous()
    b16 = torch.full_like(good, float("nan"))
    flags = torch.zeros(P, dtype=torch.int32, device="cuda")
    C = torch.full((m, n), float("nan"), device="cuda")
    io = poas.GemmIO(m=m, n=n, k=k, a16_dev=d["A16"].data_ptr(), lda16_dev=d["A16"].shape[1],
                     b16_dev=b16.data_ptr(), ldb16_dev=np_, c_dev=C.data_ptr(), ldc_dev=n,
                     resident=1, b_panels=P, b_flags=flags.data_ptr(), b_epoch=3)
    ex = poas.Executor(units)
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        torch.cuda._sleep(1_000_000)
        for p in range(P):
            b16[p].copy_(good[p])
            poas.signal_flag(flags[p:p + 1].data_ptr(), 3, s.cuda_stream)
    ex.execute(sched_text, io, 1)
    torch.cuda.synchronize()
    exp = oracle.expected_c(sched, d["A"], d["B"], {"gpu0.tc": 2})
    assert oracle.rel_frobenius(C.cpu().numpy(), exp) <= TOL


@pytest.mark.timeout(300)
@pytest.mark.parametrize("grid", ["aligned", "ragged", "aligned_n_not4", "aligned_1sm"])
@pytest.mark.parametrize("link", ["bf16", "fp32"])
@pytest.mark.parametrize("epi", [None, "8"])
def test_overlapped_grid_ragged(torch_cuda, poas, monkeypatch, link, grid, epi):
    """Overlapped execution of a hand-made 3 x 3 grid of blocks (ragged row
    parts and column panels, the tiles of an "overlap" schedule): A parts
    and B panels interleaved host->device, each block's C back as soon as it
    is computed -- every element of C exact. 16-bit link + 256-aligned grid:
    ONE streamed tensor launch (producers wait on per-item flags, the
    copy-out on per-block flags); otherwise one GEMM per block.
    "aligned_n_not4": C's pitch (n = 1002) is not a TMA pitch, so the
    streamed launch writes C with direct stores and must still raise every
    block flag; "aligned_1sm": a one-SM budget cannot run the pair kernel, so
    the streamed launch is not used (both used to hang).
    epi = "8": the streamed launch with 8 epilogue warps per CTA (16 block
    arrivals per tile)."""
    import oracle

    if epi:
        if link != "bf16":
            pytest.skip("the epilogue-warp choice is the streamed launch's")
        monkeypatch.setenv("POAS_TC_EPI", epi)

    torch = torch_cuda
    elem = 2 if link == "bf16" else 4
    sms = 1 if grid == "aligned_1sm" else 16
    units = f"gpu0.tc=xpu:dev=0:sms={sms}:dtype=bf16:elem={elem}:link=pcie:probe=512-2048"
    m, n, k = 1000, (1002 if grid == "aligned_n_not4" else 1000), 520
    profile = poas.profile_machine(units, PROF, True)
    sched = json.loads(poas.plan_policy(profile, m, n, k, "overlap"))
    parts, panels = {"aligned": ([512, 256, 232], [256, 512, 232]),
                     "aligned_1sm": ([512, 256, 232], [256, 512, 232]),
                     "aligned_n_not4": ([512, 256, 232], [256, 512, 234]),
                     "ragged": ([384, 384, 232], [256, 256, 488])}[grid]
    sched["devices"][0]["tiles"] = [{"m": r, "k": k, "n": w} for r in parts for w in panels]
    sched_text = poas.schedule_roundtrip(json.dumps(sched))
    d = operands(torch, poas, m, n, k)
    hC = torch.full((m, n), float("nan")).pin_memory()
    io = poas.GemmIO(m=m, n=n, k=k, a_host=d["hA"].data_ptr(), lda_host=k, b_host=d["hB"].data_ptr(),
                     ldb_host=n, c_host=hC.data_ptr(), ldc_host=n, resident=0)
    if link == "bf16":
        hA16 = d["A16"][:, :k].cpu().contiguous().pin_memory()
        hB16 = d["B16"][:, :n].cpu().contiguous().pin_memory()
        io.a16_host, io.lda16_host, io.b16_host, io.ldb16_host = hA16.data_ptr(), k, hB16.data_ptr(), n
    ex = poas.Executor(units + ";overlap=1")
    rep = ex.execute(sched_text, io, 2)
    exp = oracle.expected_c(sched, d["A"], d["B"], {"gpu0.tc": 2})
    got = hC.numpy()
    assert not np.isnan(got).any()
    assert oracle.rel_frobenius(got, exp) <= TOL
    assert rep["devices"][0].get("overlapped") is True
    if link == "bf16" and grid == "aligned":
        # pipelined repeats (one streamed unit): repeat r+1's copies start
        # beside r's copy-out tail, C double-buffered -- every repeat exact
        exp_host = hC.clone()
        ex_p = poas.Executor(units + ";overlap=1;pipeline=1")
        for reps in (1, 2, 5):
            hC.fill_(float("nan"))
            rep = ex_p.execute(sched_text, io, reps)
            assert oracle.rel_frobenius(hC.numpy(), exp) <= TOL, reps
            assert torch.equal(hC, exp_host), reps
            assert rep["repeats"] == reps and rep["measured_makespan"] > 0
        # new host operands between runs (odd repeats land in the second
        # staging set): 2 x A is exact in bf16 and in the fp32 sums, so every
        # run must give exactly 2 x C -- nothing stale from either set
        hA16_2 = (hA16.float() * 2).bfloat16().contiguous().pin_memory()
        io.a16_host = hA16_2.data_ptr()
        for reps in (2, 3):
            hC.fill_(float("nan"))
            ex_p.execute(sched_text, io, reps)
            assert torch.equal(hC, exp_host * 2), reps
        io.a16_host = hA16.data_ptr()
        hC.fill_(float("nan"))
        ex_p.execute(sched_text, io, 4)
        assert torch.equal(hC, exp_host)


def test_fused_link_unit_profile(torch_cuda, poas):
    """link=fused (a tensor unit whose operand stream is inside its probed
    GEMM): the profile's bandwidth is the nominal 1 PB/s, so the plan's copy
    phases are ~0 and its prediction is the compute model alone; a resident
    run through it is exact."""
    import oracle

    torch = torch_cuda
    units = ("gpu0.tc=xpu:dev=0:sms=16:dtype=bf16:elem=2:link=fused:probe=512-1024;"
             "gpu0.simt=gpu:dev=0:sms=2:exclusive=1:elem=4:link=hbm:probe=128-256")
    prof = poas.profile_machine(units, "probes=3,repetitions=2,bandwidth_payload=4194304", True, retries=2)
    bw = {}
    cur = None
    for line in prof.splitlines():
        p = line.split()
        if len(p) == 2 and p[0] == "device":
            cur = p[1]
        elif len(p) == 2 and p[0] == "bandwidth":
            bw[cur] = float(p[1])
    assert bw["gpu0.tc"] == pytest.approx(1e15, rel=1e-6)
    assert 1e9 < bw["gpu0.simt"] < 1e13
    m, n, k = 1024, 768, 512
    s = json.loads(poas.plan_policy(prof, m, n, k, "best-subset"))
    tc = [d for d in s["devices"] if d["id"] == "gpu0.tc"][0]
    assert tc["rows"] > 0
    ci, co = tc["copy_in"], tc["copy_out"]
    assert ci[1] - ci[0] < 1e-7 and co[1] - co[0] < 1e-7
    A, B = oracle.fill_uniform(m, k, 3), oracle.fill_uniform(k, n, 4)
    a16 = torch.from_numpy(A).cuda().bfloat16()
    b16 = torch.from_numpy(B).cuda().bfloat16()
    a32 = torch.from_numpy(A).cuda()
    b32 = torch.from_numpy(B).cuda()
    C = torch.full((m, n), float("nan"), device="cuda")
    io = poas.GemmIO(m=m, n=n, k=k, a_dev=a32.data_ptr(), lda_dev=k, b_dev=b32.data_ptr(), ldb_dev=n,
                     a16_dev=a16.data_ptr(), lda16_dev=k, b16_dev=b16.data_ptr(), ldb16_dev=n,
                     c_dev=C.data_ptr(), ldc_dev=n, resident=1)
    poas.Executor(units).execute(json.dumps(s), io, 1)
    torch.cuda.synchronize()
    ref = oracle.expected_c(s, A, B, {"gpu0.tc": 2, "gpu0.simt": 0})
    assert oracle.rel_frobenius(C.cpu().numpy(), ref) <= 2e-5
