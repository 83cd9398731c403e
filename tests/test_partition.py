"""The planner's SM-partition choice (poas_b200_plan_partitions, B200
extension): one GPU's SMs between its tensor unit and its CUDA-core unit,
each candidate budget planned through the POAS pipeline on a profile whose
GPU units are rescaled by their SM counts (csrc/planner/policy.cpp)."""
import json

import pytest

from conftest import GOLDEN

N = 16384
# Two regimes: the measured B200 shape (tensor cores ~9 TFLOP/s per SM, CUDA
# cores ~0.4 TFLOP/s per SM) and a synthetic machine whose CUDA cores are
# faster per SM than its tensor cores.


def _profile(tc_slope, simt_slope, simt_bw=1.07e11):
    text = (GOLDEN / "profiles" / "b200_like.profile").read_text()
    out, cur = [], None
    for line in text.splitlines():
        parts = line.split()
        if len(parts) == 2 and parts[0] == "device":
            cur = parts[1]
        if cur == "gpu0.tc" and parts[:1] == ["slope"]:
            line = f"slope {tc_slope!r}"
        if cur == "gpu0.simt" and parts[:1] == ["slope"]:
            line = f"slope {simt_slope!r}"
        if cur == "gpu0.simt" and parts[:1] == ["bandwidth"]:
            line = f"bandwidth {simt_bw!r}"
        out.append(line)
    return "\n".join(out) + "\n"


def _b200(poas):
    # tensor unit (146 SMs) 1.35 PFLOP/s; CUDA-core unit (2 SMs) 0.8 TFLOP/s
    return _profile(2.0 / 1.35e15, 2.0 / 0.8e12)


def test_b200_shape_leaves_the_cuda_cores_out(poas):
    """Tensor cores are ~25x faster per SM than the CUDA cores: every SM the
    CUDA-core unit would take costs more than it adds, so the optimizer's
    choice is budget 0 (the CUDA-core unit's SMs lent to the tensor unit)."""
    prof = _b200(poas)
    out = poas.plan_partitions(prof, N, N, N, "gpu0.tc", 146, "gpu0.simt", 2, [0, 2, 4, 8, 16, 32])
    cands = out["candidates"]
    assert [c["simt_sms"] for c in cands] == [0, 2, 4, 8, 16, 32]
    assert [c["tc_sms"] for c in cands] == [148, 146, 144, 140, 132, 116]
    best = cands[out["best"]]
    assert best["simt_sms"] == 0 and "gpu0.simt" not in best["rows"]
    assert best["rows"]["gpu0.tc"] + best["rows"].get("cpu0", 0) == N
    spans = [c["makespan"] for c in cands]
    assert spans == sorted(spans)  # more CUDA-core SMs, longer makespan
    # budget 0 is the tensor unit on all 148 SMs: 146/148 of its time
    tc_only = json.loads(poas.plan_policy(prof, N, N, N, "best-subset"))["makespan"]
    assert spans[0] < tc_only


def test_unchanged_budget_reproduces_the_plain_plan(poas):
    """The candidate at the measured budgets IS the profile: same rows and
    predicted makespan as planning it directly with the same policy."""
    prof = _b200(poas)
    out = poas.plan_partitions(prof, N, N, N, "gpu0.tc", 146, "gpu0.simt", 2, [2], "best-subset")
    direct = json.loads(poas.plan_policy(prof, N, N, N, "best-subset"))
    c = out["candidates"][0]
    assert c["rows"] == {d["id"]: d["rows"] for d in direct["devices"]}
    assert c["makespan"] == pytest.approx(direct["makespan"], abs=1e-9)  # JSON keeps %.9f


def test_fast_cuda_cores_get_sms(poas):
    """A unit that is faster per SM than the tensor unit (a synthetic
    machine) is given SMs: the choice follows the model, not a fixed split."""
    # per SM: tensor 1.35e15/146 = 9.2 TFLOP/s; CUDA cores 40e12/2 = 20 TFLOP/s
    prof = _profile(2.0 / 1.35e15, 2.0 / 40e12, simt_bw=6.5e12)
    out = poas.plan_partitions(prof, N, N, N, "gpu0.tc", 146, "gpu0.simt", 2, [0, 2, 16, 64])
    cands = out["candidates"]
    best = cands[out["best"]]
    assert best["simt_sms"] == 64
    assert best["rows"]["gpu0.simt"] > best["rows"]["gpu0.tc"]
    assert cands[out["best"]]["makespan"] == min(c["makespan"] for c in cands)


def test_partition_rejects_bad_arguments(poas):
    from paper_2209_10245_b200 import PoasError

    prof = _b200(poas)
    for bad in (dict(tc_id="nope"), dict(simt_sms=0), dict(budgets=[148]), dict(budgets=[-1])):
        kw = dict(tc_id="gpu0.tc", simt_sms=2, budgets=[0, 2])
        kw.update(bad)
        with pytest.raises(PoasError):
            poas.plan_partitions(prof, N, N, N, kw["tc_id"], 146, "gpu0.simt", kw["simt_sms"], kw["budgets"])


def test_splice_unit_replaces_the_model_keeps_the_machine(poas):
    """Predict after Optimize (bench.py): a unit re-probed on its decided SM
    budget replaces its model in the machine profile; identity, priorities
    and the machine hash stay, so schedules planned from either run on the
    same executor."""
    base = _b200(poas)
    faster = _profile(2.0 / 1.37e15, 2.0 / 0.8e12)  # the tensor unit on 148 SMs
    out = poas.splice_unit(base, faster, "gpu0.tc")
    assert poas.machine_hash(out) == poas.machine_hash(base)
    assert poas.profile_roundtrip(out) == out
    tc = [ln for ln in out.split("device gpu0.tc")[1].splitlines() if ln.startswith("slope ")][0]
    assert float(tc.split()[1]) == pytest.approx(2.0 / 1.37e15, rel=1e-15)
    simt = [ln for ln in out.split("device gpu0.simt")[1].splitlines() if ln.startswith("slope ")][0]
    assert float(simt.split()[1]) == pytest.approx(2.0 / 0.8e12, rel=1e-15)
    s0 = json.loads(poas.plan_policy(base, N, N, N, "best-subset"))
    s1 = json.loads(poas.plan_policy(out, N, N, N, "best-subset"))
    assert s1["makespan"] < s0["makespan"]
    from paper_2209_10245_b200 import PoasError

    with pytest.raises(PoasError):
        poas.splice_unit(base, faster, "gpu9.tc")
