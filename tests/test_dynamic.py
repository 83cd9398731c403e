"""Dynamic scheduling (paper §3.4.2): model re-fit from
execution reports and the re-planning loop. The reference has only the
static scheduler, so these tests pin the rebuild's own contract
(csrc/include/poas/dynamic.hpp): the update rule, identity preservation,
error behaviour, and that a mis-profiled machine converges on real runs."""
import json

import numpy as np
import pytest

from conftest import GOLDEN


def _profile_fields(text):
    devs, cur = {}, None
    for line in text.splitlines():
        parts = line.split()
        if len(parts) == 2 and parts[0] == "device":
            cur = devs.setdefault(parts[1], {})
        elif cur is not None and len(parts) == 2:
            cur[parts[0]] = parts[1]
    return devs


def _fake_report(schedule, scale_compute=None, scale_copy=None):
    """An execution report with every phase measured == predicted, except
    the per-unit scale factors given."""
    scale_compute = scale_compute or {}
    scale_copy = scale_copy or {}
    devices = []
    for d in schedule["devices"]:
        tl = d["timeline"] if "timeline" in d else d
        ci = tl["copy_in"][1] - tl["copy_in"][0]
        cc = tl["compute"][1] - tl["compute"][0]
        co = tl["copy_out"][1] - tl["copy_out"][0]
        fc, fl = scale_compute.get(d["id"], 1.0), scale_copy.get(d["id"], 1.0)

        def ph(pred, f):
            return {"measured": pred * f, "predicted": pred,
                    "error_pct": 100.0 * (pred * f - pred) / (pred * f) if pred > 0 else 0.0}

        devices.append({"id": d["id"], "rows": d["rows"], "copy_in": ph(ci, fl),
                        "compute": ph(cc, fc), "copy_out": ph(co, fl)})
    return {"measured_makespan": schedule["makespan"], "predicted_makespan": schedule["makespan"],
            "makespan_error_pct": 0.0, "devices": devices}


@pytest.fixture(scope="module")
def b200_like():
    return (GOLDEN / "profiles" / "b200_like.profile").read_text()


def test_schedule_shape_for_fake_reports(poas, b200_like):
    s = json.loads(poas.plan(b200_like, 16384, 16384, 16384))
    d = s["devices"][0]
    assert "copy_in" in d and "compute" in d and "copy_out" in d, d.keys()


@pytest.mark.parametrize("alpha,expect", [(1.0, 1.5), (0.5, 1.25)])
def test_refit_scales_compute_model(poas, b200_like, alpha, expect):
    s = json.loads(poas.plan(b200_like, 16384, 16384, 16384))
    rows = {d["id"]: d["rows"] for d in s["devices"]}
    assert rows["gpu0.tc"] > 0
    rep = _fake_report(s, scale_compute={"gpu0.tc": 1.5})
    out = poas.refit_profile(b200_like, rep, alpha)
    before, after = _profile_fields(b200_like), _profile_fields(out)
    assert float(after["gpu0.tc"]["slope"]) == pytest.approx(float(before["gpu0.tc"]["slope"]) * expect,
                                                             rel=1e-15)
    assert float(after["gpu0.tc"]["intercept"]) == pytest.approx(
        float(before["gpu0.tc"]["intercept"]) * expect, rel=1e-15)
    for uid in ("cpu0", "gpu0.simt"):
        if rows[uid] > 0:
            for key in ("slope", "intercept", "bandwidth"):
                assert float(after[uid][key]) == pytest.approx(float(before[uid][key]), rel=1e-15)
    # everything but the model is as profiled: same identity, priorities, windows
    for uid in before:
        for key in ("kind", "elem_size", "priority", "ops_min", "ops_max"):
            assert after[uid].get(key) == before[uid].get(key), (uid, key)
    assert poas.machine_hash(out) == poas.machine_hash(b200_like)
    # the text is a canonical profile (round-trips byte-identically)
    assert poas.profile_roundtrip(out) == out


def test_refit_bandwidth_from_copy_phases(poas, b200_like):
    s = json.loads(poas.plan(b200_like, 16384, 16384, 16384))
    rep = _fake_report(s, scale_copy={"gpu0.tc": 2.0})
    out = _profile_fields(poas.refit_profile(b200_like, rep, 1.0))
    bw0 = float(_profile_fields(b200_like)["gpu0.tc"]["bandwidth"])
    assert float(out["gpu0.tc"]["bandwidth"]) == pytest.approx(bw0 / 2.0, rel=1e-15)
    assert float(out["gpu0.tc"]["slope"]) == pytest.approx(
        float(_profile_fields(b200_like)["gpu0.tc"]["slope"]), rel=1e-15)


def test_refit_step_is_clamped(poas, b200_like):
    s = json.loads(poas.plan(b200_like, 16384, 16384, 16384))
    out = _profile_fields(poas.refit_profile(b200_like, _fake_report(s, {"gpu0.tc": 100.0}), 1.0))
    assert float(out["gpu0.tc"]["slope"]) == pytest.approx(
        4.0 * float(_profile_fields(b200_like)["gpu0.tc"]["slope"]), rel=1e-15)


def test_refit_moves_rows_away_from_slow_unit(poas, b200_like):
    m = n = k = 16384
    s0 = json.loads(poas.plan(b200_like, m, n, k))
    r0 = {d["id"]: d["rows"] for d in s0["devices"]}
    slow = poas.refit_profile(b200_like, _fake_report(s0, {"gpu0.tc": 3.0}), 1.0)
    s1 = json.loads(poas.plan(slow, m, n, k))
    r1 = {d["id"]: d["rows"] for d in s1["devices"]}
    assert r1["gpu0.tc"] < r0["gpu0.tc"]
    assert sum(r1.values()) == m
    assert s1["machine_hash"] == s0["machine_hash"]


def test_refit_ignores_idle_units_and_zero_phases(poas, b200_like):
    s = json.loads(poas.plan(b200_like, 16384, 16384, 16384))
    rep = _fake_report(s, {d["id"]: 2.0 for d in s["devices"]})
    for d in rep["devices"]:
        if d["id"] == "gpu0.simt":
            d["rows"] = 0
        if d["id"] == "cpu0":
            d["compute"]["measured"] = 0.0
    out, before = _profile_fields(poas.refit_profile(b200_like, rep, 1.0)), _profile_fields(b200_like)
    assert out["gpu0.simt"]["slope"] == before["gpu0.simt"]["slope"]
    assert out["cpu0"]["slope"] == before["cpu0"]["slope"]


def test_refit_errors(poas, b200_like):
    from paper_2209_10245_b200 import PoasError

    s = json.loads(poas.plan(b200_like, 4096, 4096, 4096))
    rep = _fake_report(s)
    with pytest.raises(PoasError) as e:
        poas.refit_profile(b200_like, rep, 0.0)
    assert e.value.errc == "invalid_argument"
    with pytest.raises(PoasError) as e:
        poas.refit_profile(b200_like, rep, 1.5)
    assert e.value.errc == "invalid_argument"
    bad = json.loads(json.dumps(rep))
    bad["devices"][0]["id"] = "gpu9.tc"
    with pytest.raises(PoasError) as e:
        poas.refit_profile(b200_like, bad, 0.5)
    assert e.value.errc == "missing_device"
    for broken in ("{", '{"devices": 3, "measured_makespan": 1, "predicted_makespan": 1, '
                        '"makespan_error_pct": 0}', json.dumps({"devices": []})):
        with pytest.raises(PoasError) as e:
            poas.refit_profile(b200_like, broken, 0.5)
        assert e.value.errc == "parse_failure"


def test_dynamic_loop_converges_on_host_units(poas):
    """Real executions on two host CPU units whose profile is planted 8x too
    optimistic for one of them: the loop re-fits, re-plans, moves rows away
    and the prediction error shrinks; C stays exact."""
    units = "cpuA=cpu:threads=1;cpuB=cpu:threads=1"
    prof = poas.profile_machine(units, "probes=3,repetitions=3,cpu_min_side=192,cpu_max_side=448", retries=3)
    lines = []
    cur = None
    for line in prof.splitlines():
        parts = line.split()
        if len(parts) == 2 and parts[0] == "device":
            cur = parts[1]
        if cur == "cpuA" and len(parts) == 2 and parts[0] in ("slope", "intercept"):
            line = f"{parts[0]} {float(parts[1]) / 8.0!r}"
        lines.append(line)
    planted = "\n".join(lines) + "\n"
    m, n, k = 1024, 256, 256
    rng = np.random.default_rng(7)
    A = rng.uniform(-1, 1, (m, k)).astype(np.float32)
    B = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    C = np.zeros((m, n), np.float32)
    io = poas.GemmIO(m=m, n=n, k=k, a_host=A.ctypes.data, lda_host=k, b_host=B.ctypes.data,
                     ldb_host=n, c_host=C.ctypes.data, ldc_host=n, resident=0)
    ex = poas.Executor(units)
    out = ex.run_dynamic(planted, m, n, k, io, iterations=6, alpha=1.0, replan_threshold_pct=5.0)
    its = out["iterations"]
    assert len(its) == 6 and out["replans"] >= 1
    assert its[0]["replanned"] is False and any(i["replanned"] for i in its[1:])
    assert its[-1]["rows"]["cpuA"] < its[0]["rows"]["cpuA"]
    assert all(sum(i["rows"].values()) == m for i in its)
    assert abs(its[-1]["makespan_error_pct"]) < abs(its[0]["makespan_error_pct"])
    assert poas.machine_hash(out["profile"]) == poas.machine_hash(planted)
    assert out["schedule"]["machine_hash"] == ex.machine_hash
    # the returned plan is the fastest MEASURED one (the last re-plan is
    # unmeasured and a re-fit's plan can be slower than its predecessor)
    best = out["best_iteration"]
    assert its[best]["measured_makespan"] == min(i["measured_makespan"] for i in its)
    assert {d["id"]: d["rows"] for d in out["schedule"]["devices"]} == its[best]["rows"]
    assert out["last_schedule"]["machine_hash"] == ex.machine_hash
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert np.linalg.norm(C - ref) / np.linalg.norm(ref) < 2e-5


def test_dynamic_rejects_bad_arguments(poas):
    from paper_2209_10245_b200 import PoasError

    prof = (GOLDEN / "profiles" / "cpu_only.profile").read_text()
    ex = poas.Executor("cpu0=cpu:threads=1")
    io = poas.GemmIO(m=64, n=64, k=64, resident=0)
    with pytest.raises(PoasError) as e:
        ex.run_dynamic(prof, 64, 64, 64, io, iterations=0)
    assert e.value.errc == "invalid_argument"
    with pytest.raises(PoasError) as e:
        ex.run_dynamic(prof, 64, 64, 64, io, iterations=1, policy="nope")
    assert e.value.errc == "invalid_argument"


def test_refit_resident_unit_folds_link_phases_into_compute(poas, b200_like):
    """Resident operands: predicted copy phases, none measured -- the kernel
    streamed its operands while computing. The compute model moves so the
    three predicted phases add up to the measured compute; bandwidth stays."""
    s = json.loads(poas.plan(b200_like, 16384, 16384, 16384))
    rep = _fake_report(s)
    tc = [d for d in rep["devices"] if d["id"] == "gpu0.tc"][0]
    link = tc["copy_in"]["predicted"] + tc["copy_out"]["predicted"]
    assert link > 0
    whole = tc["compute"]["predicted"] + link
    for ph in ("copy_in", "copy_out"):
        tc[ph]["measured"] = 0.0
    tc["compute"]["measured"] = 0.9 * whole
    out = poas.refit_profile(b200_like, rep, 1.0)
    before, after = _profile_fields(b200_like), _profile_fields(out)
    # the same rows now predict copy-in + compute + copy-out == measured
    g = (0.9 * whole - link) / tc["compute"]["predicted"]
    for key in ("slope", "intercept"):
        assert float(after["gpu0.tc"][key]) == pytest.approx(float(before["gpu0.tc"][key]) * g,
                                                             rel=1e-12)
    assert after["gpu0.tc"]["bandwidth"] == before["gpu0.tc"]["bandwidth"]


def test_refit_resident_unit_by_finish(poas, b200_like):
    """Resident operands with the unit's finish measured: its whole timeline
    (compute and the modelled operand stream) scales by the finish ratio
    (launch latency between t0 and the kernel is part of it), so the
    re-planned finish matches the measurement."""
    s = json.loads(poas.plan(b200_like, 16384, 16384, 16384))
    rep = _fake_report(s)
    tc = [d for d in rep["devices"] if d["id"] == "gpu0.tc"][0]
    sd = [d for d in s["devices"] if d["id"] == "gpu0.tc"][0]
    for ph in ("copy_in", "copy_out"):
        tc[ph]["measured"] = 0.0
    fin_pred = sd["copy_out"][1]
    tc["finish"] = {"measured": fin_pred + 0.0004, "predicted": fin_pred, "error_pct": 0.0}
    out = poas.refit_profile(b200_like, rep, 1.0)
    before, after = _profile_fields(b200_like), _profile_fields(out)
    g = (fin_pred + 0.0004) / fin_pred  # the whole timeline scales by the finish ratio
    for key in ("slope", "intercept"):
        assert float(after["gpu0.tc"][key]) == pytest.approx(float(before["gpu0.tc"][key]) * g, rel=1e-9)
    assert float(after["gpu0.tc"]["bandwidth"]) == pytest.approx(float(before["gpu0.tc"]["bandwidth"]) / g,
                                                                 rel=1e-9)
    # re-planned with the same rows, the unit's predicted finish is the measurement
    s2 = json.loads(poas.plan(out, 16384, 16384, 16384))
    sd2 = [d for d in s2["devices"] if d["id"] == "gpu0.tc"][0]
    if sd2["rows"] == sd["rows"]:
        assert sd2["copy_out"][1] == pytest.approx(fin_pred + 0.0004, rel=1e-6)
