"""Plan parity: the B200 planner (libpoas_b200.so) against the reference
planner (oracle/_ref, compiled from /root/reference/proj/src) and against the
committed golden fixtures made from it (tools/make_golden.py).

north_star: "Partition plans must be bit-exact given the same profiles" --
checked as byte-identical format_schedule output (reference
proj/src/scheduler.cpp:147-183) plus %.17g-identical WorkloadSplit fields.
"""
import hashlib
import json
import random

import pytest

from conftest import GOLDEN


def _fmt(x):
    return repr(float(x))


def random_profile(rng: random.Random, n_dev: int, with_cpu: bool, bus: bool) -> str:
    """Random machine in (and around) the planner's operating regime: the
    reference's random_accel_machine (proj/tests/support.hpp:103-126) widened
    with cpu units, B200-like tensor/SIMT speed ratios and private links."""
    lines = ["poas-profile v1", "", f"bus {'true' if bus else 'false'}"]
    kinds = []
    if with_cpu:
        kinds.append("cpu")
    while len(kinds) < n_dev:
        kinds.append(rng.choice(["gpu", "xpu"]))
    prios = list(range(n_dev))
    rng.shuffle(prios)
    for i, kind in enumerate(kinds):
        regime = rng.random()
        if kind == "cpu":
            slope = rng.uniform(5e-13, 3e-12)
        elif regime < 0.5:
            slope = rng.uniform(8e-14, 4e-13)  # reference random_accel_machine
        else:
            slope = rng.uniform(1e-15, 5e-14)  # B200-like tensor / SIMT
        icpt = rng.choice([0.0, rng.uniform(1e-6, 1e-2)])
        bw = 0.0 if kind == "cpu" else rng.choice([rng.uniform(16e9, 64e9), rng.uniform(5e11, 7e12)])
        elem = 4 if kind == "cpu" else rng.choice([2, 4])
        lo = rng.choice([256, 500, 1000, 2048, 3000])
        hi = lo * rng.choice([1, 2, 3, 4, 6])
        lines += ["", f"device {kind}{i}", f"kind {kind}", f"slope {_fmt(slope)}",
                  f"intercept {_fmt(icpt)}", f"bandwidth {_fmt(bw)}", f"elem_size {elem}",
                  f"priority {prios[i]}"]
        if kind == "xpu":
            lines.append(f"align {rng.choice([1, 8, 8, 16])}")
        if kind == "cpu":
            lines.append("cache_bytes 33554432")
        lines += [f"ops_min {lo ** 3}", f"ops_max {hi ** 3}"]
    return "\n".join(lines) + "\n"


def random_dims(rng: random.Random):
    r = rng.random()
    if r < 0.4:  # reference random_large_dims (support.hpp:128-135)
        return rng.randint(20000, 60000), rng.randint(8000, 20000), rng.randint(8000, 20000)
    if r < 0.7:  # B200 shapes
        s = rng.choice([1024, 2048, 4096, 8192, 16384])
        return rng.choice([s, 4 * s, 8 * s]), s, s
    return rng.randint(1, 5000), rng.randint(1, 5000), 8 * rng.randint(1, 700)


def both(fn_ours, fn_ref, *args):
    """(ok, value) from each side; errors compared by errc code."""
    import oracle
    from paper_2209_10245_b200 import PoasError

    try:
        a = ("ok", fn_ours(*args))
    except PoasError as e:
        a = ("err", e.code)
    try:
        b = ("ok", fn_ref(*args))
    except oracle.OracleError as e:
        b = ("err", e.code)
    return a, b


def test_golden_plans_match(poas):
    cases = json.loads((GOLDEN / "plans.json").read_text())
    profiles = {p.stem: p.read_text() for p in (GOLDEN / "profiles").glob("*.profile")}
    for c in cases:
        prof = profiles[c["profile"]]
        if c["error"] is not None:
            with pytest.raises(Exception):
                poas.plan(prof, c["m"], c["n"], c["k"])
            continue
        sched = poas.plan(prof, c["m"], c["n"], c["k"])
        assert hashlib.sha256(sched.encode()).hexdigest() == c["schedule_sha256"], c["profile"]
        if c["schedule"] is not None:
            assert sched == c["schedule"]
        assert poas.solve_split(prof, c["m"], c["n"], c["k"]) == c["split"]


def test_golden_profiles_roundtrip(poas):
    for p in (GOLDEN / "profiles").glob("*.profile"):
        text = p.read_text()
        assert poas.profile_roundtrip(text) == text


def test_appendix_d_cpu_only_schedule(poas):
    """the CPU-only 2048^3 plan, the complete file."""
    prof = (GOLDEN / "profiles" / "cpu_only.profile").read_text()
    sched = json.loads(poas.plan(prof, 2048, 2048, 2048))
    d = sched["devices"][0]
    assert sched["machine_hash"] == "f0950b5f8e921f86"
    assert d["rows"] == 2048 and len(d["tiles"]) == 4
    assert all(t == {"m": 1024, "k": 1024, "n": 2048} for t in d["tiles"])
    assert d["compute"] == [0.0, 0.017679869]
    assert sched["makespan"] == 0.017679869


@pytest.mark.parametrize("seed", range(8))
def test_random_plans_byte_identical(poas, ref, seed):
    """>= 10k random instances overall (8 seeds x 1300 + the rest)."""
    rng = random.Random(1000 + seed)
    n_cmp = 0
    for _ in range(1300):
        nd = rng.randint(1, 4)
        prof = random_profile(rng, nd, with_cpu=rng.random() < 0.5, bus=rng.random() < 0.8)
        m, n, k = random_dims(rng)
        a, b = both(poas.plan, ref.plan, prof, m, n, k)
        assert a == b, (prof, m, n, k)
        s1, s2 = both(poas.solve_split, ref.solve_split, prof, m, n, k)
        assert s1 == s2, (prof, m, n, k)
        n_cmp += 1
    assert n_cmp == 1300


def test_b200_like_profile_matches_survey(poas, ref):
    """SURVEY.md Appendix B, illustrative B200-like profile at 16384^3: rows
    CPU 15 / SIMT 641 / TC 15728 after the reference's residue and shave
    rules (the 8.553 ms schedule)."""
    prof = (GOLDEN / "profiles" / "b200_like.profile").read_text()
    s = json.loads(poas.plan(prof, 16384, 16384, 16384))
    rows = {d["id"]: d["rows"] for d in s["devices"]}
    assert rows == {"gpu0.tc": 15728, "gpu0.simt": 641, "cpu0": 15}
    assert abs(s["makespan"] - 0.008553) < 1e-6
    assert poas.plan(prof, 16384, 16384, 16384) == ref.plan(prof, 16384, 16384, 16384)


def test_policy_reference_is_the_reference_and_best_subset_never_worse(poas, ref):
    """The default planner policy is byte-identical to the reference; the
    opt-in best-subset policy (B200 extension) never predicts a longer
    makespan, and on the survey's B200-like profile it recovers the
    no-CPU plan (8.553 ms -> 6.448 ms)."""
    prof = (GOLDEN / "profiles" / "b200_like.profile").read_text()
    s = json.loads(poas.plan_policy(prof, 16384, 16384, 16384, "best-subset"))
    assert {d["id"]: d["rows"] for d in s["devices"]} == {"gpu0.tc": 15736, "gpu0.simt": 648, "cpu0": 0}
    assert abs(s["makespan"] - 0.006448) < 1e-6
    rng = random.Random(99)
    for _ in range(150):
        nd = rng.randint(1, 4)
        prof = random_profile(rng, nd, with_cpu=rng.random() < 0.5, bus=rng.random() < 0.8)
        m, n, k = random_dims(rng)
        a, b = both(lambda *x: poas.plan_policy(*x, "reference"), ref.plan, prof, m, n, k)
        assert a == b
        if a[0] != "ok":
            continue
        best = json.loads(poas.plan_policy(prof, m, n, k, "best-subset"))
        assert best["makespan"] <= json.loads(a[1])["makespan"] + 1e-9
        assert sum(d["rows"] for d in best["devices"]) == m
        assert best["machine_hash"] == json.loads(a[1])["machine_hash"]


def test_standalone_plans(poas, ref):
    for name in ("mach2_exact", "mach2_seed7", "b200_like"):
        prof = (GOLDEN / "profiles" / f"{name}.profile").read_text()
        ids = [ln.split()[1] for ln in prof.splitlines() if ln.startswith("device ")]
        for dev in ids:
            for dims in [(16003, 4000, 4000), (16000, 16000, 16000), (8192, 8192, 8192)]:
                a, b = both(poas.plan_standalone, ref.plan_standalone, prof, dev, *dims)
                assert a == b


def test_oracle_grid_search_parity(poas, ref):
    rng = random.Random(7)
    for _ in range(40):
        nd = rng.randint(1, 3)
        prof = random_profile(rng, nd, with_cpu=rng.random() < 0.5, bus=rng.random() < 0.7)
        m, n, k = random_dims(rng)
        res = rng.choice([50, 200, 1000])
        for par in (True, False):
            a, b = both(poas.oracle_grid_search, ref.oracle_grid_search, prof, m, n, k, res, par)
            assert a == b
        # parallel == serial (reference proj/tests/test_optimizer.cpp:168-180)
        a = both(poas.oracle_grid_search, ref.oracle_grid_search, prof, m, n, k, res, True)[0]
        c = both(poas.oracle_grid_search, ref.oracle_grid_search, prof, m, n, k, res, False)[0]
        assert a == c


def test_tile_plan_parity(poas, ref):
    rng = random.Random(11)
    for _ in range(400):
        nd = rng.randint(1, 3)
        prof = random_profile(rng, nd, with_cpu=rng.random() < 0.5, bus=True)
        m, n, k = random_dims(rng)
        cuts = sorted(rng.randint(0, m) for _ in range(nd - 1))
        rows = [b - a for a, b in zip([0] + cuts, cuts + [m])]
        a, b = both(poas.build_tile_plan, ref.build_tile_plan, prof, m, n, k, rows)
        assert a == b, (prof, m, n, k, rows)


def test_fit_linear_parity(poas, ref):
    rng = random.Random(3)
    for _ in range(300):
        cnt = rng.randint(2, 30)
        ops = [rng.choice([rng.randint(1, 10**6), rng.randint(10**9, 10**14)]) for _ in range(cnt)]
        slope, icpt = rng.uniform(1e-15, 1e-11), rng.uniform(-1e-3, 1e-2)
        secs = [max(1e-9, slope * o + icpt) * (1 + rng.uniform(-0.05, 0.05)) for o in ops]
        a, b = both(poas.fit_linear, ref.fit_linear, ops, secs)
        assert a == b


def test_simplex_parity(poas, ref):
    rng = random.Random(5)
    for _ in range(300):
        nv = rng.randint(1, 8)
        ne, ng = rng.randint(0, 3), rng.randint(0, 4)
        obj = [rng.uniform(-1, 2) for _ in range(nv)]
        eqa = [[rng.choice([0.0, rng.uniform(-2, 3)]) for _ in range(nv)] for _ in range(ne)]
        eqb = [rng.uniform(0, 5) for _ in range(ne)]
        gea = [[rng.choice([0.0, rng.uniform(-2, 3)]) for _ in range(nv)] for _ in range(ng)]
        geb = [rng.uniform(-2, 5) for _ in range(ng)]
        # keep problems bounded: add sum(x) <= 10 as -sum(x) >= -10
        gea.append([-1.0] * nv)
        geb.append(-10.0)
        a, b = both(poas.solve_simplex, ref.solve_simplex, obj, eqa, eqb, gea, geb)
        assert a == b


def test_transfer_bytes_and_hash_parity(poas, ref):
    rng = random.Random(9)
    for _ in range(200):
        prof = random_profile(rng, rng.randint(1, 4), with_cpu=True, bus=rng.random() < 0.5)
        assert poas.machine_hash(prof) == ref.machine_hash(prof)
        m, n, k = random_dims(rng)
        dev = [ln.split()[1] for ln in prof.splitlines() if ln.startswith("device ")][-1]
        ops = rng.choice([0, n * k * rng.randint(1, m), n * k * rng.randint(1, m) + 1])
        a, b = both(poas.transfer_bytes, ref.transfer_bytes, prof, dev, ops, m, n, k)
        assert a == b


def test_schedule_roundtrip_and_rejection_parity(poas, ref):
    prof = (GOLDEN / "profiles" / "mach2_seed7.profile").read_text()
    good = poas.plan(prof, 16000, 16000, 16000)
    assert poas.schedule_roundtrip(good) == good == ref.schedule_roundtrip(good)
    bad = [
        good.replace('"version": 1', '"version": 2'),
        good.replace('"rows": 11992', '"rows": -1'),
        good.replace('"makespan"', '"makespanx"'),
        good.replace('{"m": 1999', '{"m": 0', 1),
        good.replace('"priority": 1', '"priority": 0'),
        good[:-3],
        good.replace('"dims": {', '"dims": {"x": 1, '),
        good.replace('"version": 1', '"version": 1.0'),
        good.replace("[0.000000000, 0.056872635]", "[0.056872635, 0.0]"),
        good.replace('"id": "xpu0"', '"id": ""'),
        '{"version": 1}',
        "",
        "[]",
    ]
    for text in bad:
        a, b = both(poas.schedule_roundtrip, ref.schedule_roundtrip, text)
        assert a[0] == b[0] == "err", text[:80]
        assert a[1] == b[1] == 5  # parse_failure (or invalid_argument via validate_dims)


def test_profile_parse_rejection_parity(poas, ref):
    prof = (GOLDEN / "profiles" / "mach2_exact.profile").read_text()
    variants = [
        prof.replace("poas-profile v1", "poas-profile v2"),
        prof.replace("kind gpu", "kind tpu"),
        prof.replace("slope 1.1242270938729623e-13", "slope abc"),
        prof.replace("align 8", "align 8\nalign 8"),
        prof.replace("cache_bytes 33554432", "cache_bytes -1"),
        prof.replace("priority 1", "priority 0"),
        prof.replace("device gpu0", " device gpu0"),
        prof.replace("bus true", "bus maybe"),
        prof + "\nweird block\n",
        prof.replace("ops_min 1000000000\n", ""),
        prof.replace("elem_size 2", "elem_size 2 "),
        prof.replace("\r", "") .replace("\n", "\r\n"),
    ]
    for text in variants:
        a, b = both(poas.profile_roundtrip, ref.profile_roundtrip, text)
        assert a == b, text[:200]
