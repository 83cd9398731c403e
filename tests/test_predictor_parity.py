"""Predict parity: the product's probing + fitting pipeline (run_compute_probes,
run_bandwidth_probe, fit_machine, priority ranking, tile windows,
format_profile -- csrc/planner/profile.cpp behind poas_b200_profile_backends)
against the reference's (proj/src/profiler.cpp:25-135, driven by
profile_machine, proj/src/simulator.cpp:53-74).

Pin: the reference's synthetic backends (noise from the seed) are run by the
reference's own profiler inside oracle/_ref, which records every measurement
in call order (oracle/ref_shim.cpp ref_probe_trace). Those measurements are
replayed through the product's profiler via C callbacks -- the replay also
checks that the product asks for the same side (or payload) at every call --
and the profile text must be byte-identical to the reference's
ref_profile_synthetic for the same config and seed.

The known answers of proj/tests/test_profiler.cpp (which does not compile
here: no doctest) are re-expressed below against the product.
"""
import random

import pytest

from conftest import GOLDEN

ORACLE_REF = pytest.importorskip("oracle").REF_SO


def _need_ref():
    if not ORACLE_REF.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference)")


def _replay_devices(trace):
    """Product backends returning the reference's recorded measurements."""
    devs = []
    for d in trace["devices"]:
        gemm, xfer = list(d["gemm"]), list(d["transfer"])
        pos = {"g": 0, "t": 0}

        def tg(side, gemm=gemm, pos=pos):
            want, t = gemm[pos["g"]]
            assert side == want, f"probe side {side}, reference probed {want}"
            pos["g"] += 1
            return t

        def tt(nbytes, xfer=xfer, pos=pos):
            want, t = xfer[pos["t"]]
            assert nbytes == want, f"payload {nbytes}, reference used {want}"
            pos["t"] += 1
            return t

        devs.append({"id": d["id"], "kind": d["kind"], "elem_size": d["elem_size"],
                     "align": d["align"], "cache_bytes": d["cache_bytes"],
                     "priority": None if d["priority"] < 0 else d["priority"],
                     "time_gemm": tg, "time_transfer": tt if d["kind"] != "cpu" else None,
                     "_pos": pos, "_n": (len(gemm), len(xfer))})
    return devs


def _profiling_str(p):
    return ",".join(f"{k}={v}" for k, v in p.items())


def _replay(poas, trace):
    devs = _replay_devices(trace)
    text = poas.profile_backends(devs, _profiling_str(trace["profiling"]), trace["bus"])
    for d in devs:  # every recorded measurement consumed, none extra
        assert (d["_pos"]["g"], d["_pos"]["t"]) == d["_n"], d["id"]
    return text


def random_machine_config(rng: random.Random) -> str:
    """A random "poas-machine v1" (proj/src/machine_config.cpp format):
    1-4 devices, noisy laws, random probe grids, all-or-none priorities."""
    n = rng.randint(1, 4)
    kinds = [rng.choice(["cpu", "gpu", "xpu"]) for _ in range(n)]
    fixed = rng.random() < 0.3
    prios = list(range(n))
    rng.shuffle(prios)
    cmin = rng.choice([16, 100, 500, 1000])
    amin = rng.choice([64, 1000, 3000, 8192])
    lines = ["poas-machine v1", "", f"bus {rng.choice(['true', 'false'])}", "", "profiling",
             f"probes {rng.randint(2, 40)}", f"repetitions {rng.randint(1, 6)}",
             f"cpu_min_side {cmin}", f"cpu_max_side {cmin * rng.choice([1, 2, 3]) + rng.randint(0, 50)}",
             f"accel_min_side {amin}", f"accel_max_side {amin * rng.choice([1, 2, 4]) + rng.randint(0, 50)}",
             f"bandwidth_payload {rng.choice([1 << 20, 64 << 20, 256 << 20])}"]
    for i, kind in enumerate(kinds):
        slope = {"cpu": rng.uniform(5e-13, 3e-12), "gpu": rng.uniform(1e-14, 4e-13),
                 "xpu": rng.uniform(5e-16, 5e-14)}[kind]
        lines += ["", f"device {kind}{i}", f"kind {kind}", f"true_slope {slope!r}",
                  f"true_intercept {rng.choice([0.0, rng.uniform(1e-6, 1e-2)])!r}"]
        if kind != "cpu":
            lines.append(f"true_bandwidth {rng.uniform(1e10, 8e12)!r}")
        lines += [f"elem_size {4 if kind != 'xpu' else rng.choice([2, 4])}",
                  f"noise {rng.choice([0.0, rng.uniform(0.0, 0.2)])!r}", "drift 0"]
        if fixed:
            lines.append(f"priority {prios[i]}")
        if kind == "xpu":
            lines.append(f"align {rng.choice([1, 8, 16])}")
        if kind == "cpu":
            lines.append(f"cache_bytes {rng.choice([33554432, 268435456])}")
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("seed", [0, 1, 7, 20261017])
def test_mach2_profile_bytes_match_reference(poas, seed):
    """The reference fixture machine (noise 0) and the same machine with
    noise: replayed through the product, identical profile bytes."""
    import oracle

    _need_ref()
    cfg = (GOLDEN / "mach2.cfg").read_text()
    if seed:
        cfg = cfg.replace("noise 0\n", "noise 0.05\n")
    ref = oracle.ref.profile_synthetic(cfg, seed)
    assert _replay(poas, oracle.ref.probe_trace(cfg, seed)) == ref


def test_random_configs_profile_bytes_match_reference(poas):
    """1000+ random machines: run_compute_probes' side schedule (llround,
    clamping, de-duplication), the mean over repetitions, the bandwidth
    probe, fit_linear, windows and priority ranking -- byte-identical."""
    import oracle
    from paper_2209_10245_b200 import PoasError

    _need_ref()
    rng = random.Random(20261017)
    ok = errs = 0
    for case in range(1300):
        cfg = random_machine_config(rng)
        seed = rng.getrandbits(64)
        try:
            ref = ("ok", oracle.ref.profile_synthetic(cfg, seed))
        except oracle.OracleError as e:
            ref = ("err", e.code)
        if ref[0] == "err":  # config the reference rejects: the product must too
            trace = None
            try:
                trace = oracle.ref.probe_trace(cfg, seed)
            except oracle.OracleError:
                errs += 1
                continue
            with pytest.raises(PoasError) as ei:
                _replay(poas, trace)
            assert ei.value.code == ref[1], (case, cfg)
            errs += 1
            continue
        assert _replay(poas, oracle.ref.probe_trace(cfg, seed)) == ref[1], (case, cfg)
        ok += 1
    assert ok >= 1000, (ok, errs)


# ---- proj/tests/test_profiler.cpp, re-expressed against the product -------
def _law(slope, intercept, bandwidth, calls=None):
    def tg(side):
        if calls is not None:
            calls.append(side)
        ops = float(side) * float(side) * float(side)
        return slope * ops + intercept

    def tt(nbytes):
        return float(nbytes) / bandwidth

    return tg, (tt if bandwidth > 0 else None)


def _profile(poas, devs, profiling="", bus=True):
    return poas.profile_backends(devs, profiling, bus)


def _parse(text):
    out, cur = {}, None
    for line in text.splitlines():
        if line.startswith("device "):
            cur = out.setdefault(line.split()[1], {})
        elif cur is not None and " " in line:
            k, v = line.split(" ", 1)
            cur[k] = v
    return out


def test_compute_probes_cover_range_unique_sides(poas):
    """test_profiler.cpp:52-70: 30 unique integer sides 1000..2000; a range
    narrower than the probe count collapses to its integer sides."""
    calls = []
    tg, _ = _law(1e-12, 0.001, 0, calls)
    _profile(poas, [{"id": "cpu0", "kind": "cpu", "elem_size": 4, "time_gemm": tg}],
             "probes=30,repetitions=5,cpu_min_side=1000,cpu_max_side=2000")
    sides = list(dict.fromkeys(calls))
    assert len(calls) == 150 and len(sides) == 30
    assert sides[0] == 1000 and sides[-1] == 2000
    assert all(calls.count(s) == 5 for s in sides)
    calls.clear()
    _profile(poas, [{"id": "cpu0", "kind": "cpu", "elem_size": 4, "time_gemm": tg}],
             "probes=30,repetitions=5,cpu_min_side=10,cpu_max_side=12")
    assert list(dict.fromkeys(calls)) == [10, 11, 12]


def test_probes_reject_non_positive_time(poas):
    """test_profiler.cpp:72-80: a backend reporting 0 s -> non_positive_time."""
    from paper_2209_10245_b200 import PoasError

    with pytest.raises(PoasError) as ei:
        _profile(poas, [{"id": "g", "kind": "gpu", "elem_size": 4, "time_gemm": lambda s: 0.0}],
                 "probes=5,repetitions=1,accel_min_side=100,accel_max_side=200")
    assert ei.value.errc == "non_positive_time"
    with pytest.raises(PoasError) as ei:
        _profile(poas, [{"id": "g", "kind": "gpu", "elem_size": 4, "time_gemm": lambda s: 1e-3,
                         "time_transfer": lambda b: -1.0}], "probes=5,repetitions=1")
    assert ei.value.errc == "non_positive_time"


def test_bandwidth_probe_is_payload_over_mean_time(poas):
    """test_profiler.cpp:82-87: 32e9 B/s law -> bandwidth 32e9 (1e-12);
    payloads under 1 MiB are rejected."""
    from paper_2209_10245_b200 import PoasError

    tg, tt = _law(1e-13, 0.0, 32e9)
    prof = _parse(_profile(poas, [{"id": "g", "kind": "gpu", "elem_size": 4, "time_gemm": tg,
                                   "time_transfer": tt}], f"bandwidth_payload={256 << 20}"))
    assert float(prof["g"]["bandwidth"]) == pytest.approx(32e9, rel=1e-12)
    with pytest.raises(PoasError) as ei:
        _profile(poas, [{"id": "g", "kind": "gpu", "elem_size": 4, "time_gemm": tg,
                         "time_transfer": tt}], "bandwidth_payload=1024")
    assert ei.value.errc == "invalid_argument"


def test_fit_machine_recovers_laws_and_ranks(poas):
    """test_profiler.cpp:89-119: noise-free slopes to 1e-9, priorities
    xpu0=0 / gpu0=1 / cpu0=2, windows = the probe ranges' cubes."""
    truth = {"cpu0": ("cpu", 1.4492753623188405e-12, 0.002, 0, 4),
             "gpu0": ("gpu", 1.1242270938729624e-13, 0.005, 31.75e9, 4),
             "xpu0": ("xpu", 3.7209302325581396e-14, 0.005, 15.75e9, 2)}
    devs = []
    for did, (kind, s, c, bw, e) in truth.items():
        tg, tt = _law(s, c, bw)
        devs.append({"id": did, "kind": kind, "elem_size": e, "time_gemm": tg, "time_transfer": tt,
                     "align": 8, "cache_bytes": 32 << 20})
    prof = _parse(_profile(poas, devs))
    for did, (_, s, _, _, _) in truth.items():
        assert float(prof[did]["slope"]) == pytest.approx(s, rel=1e-9)
    assert [prof[x]["priority"] for x in ("xpu0", "gpu0", "cpu0")] == ["0", "1", "2"]
    assert prof["cpu0"]["ops_min"] == "1000000000" and prof["cpu0"]["ops_max"] == "8000000000"
    assert prof["xpu0"]["ops_min"] == "27000000000" and prof["xpu0"]["ops_max"] == "216000000000"


def test_fixed_priorities_all_or_nothing(poas):
    """test_profiler.cpp:121-136: fixed priorities override throughput
    order; fixing only some of them is an error."""
    from paper_2209_10245_b200 import PoasError

    ga, ta = _law(1e-13, 0.001, 16e9)
    gb, tb = _law(2e-13, 0.001, 16e9)
    devs = [{"id": "a", "kind": "gpu", "elem_size": 4, "time_gemm": ga, "time_transfer": ta, "priority": 1},
            {"id": "b", "kind": "gpu", "elem_size": 4, "time_gemm": gb, "time_transfer": tb, "priority": 0}]
    prof = _parse(_profile(poas, devs))
    assert prof["a"]["priority"] == "1" and prof["b"]["priority"] == "0"
    devs[1]["priority"] = None
    with pytest.raises(PoasError) as ei:
        _profile(poas, devs)
    assert ei.value.errc == "invalid_argument"
