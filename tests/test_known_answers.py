"""Known-answer tests of the reference suite,
re-expressed against the B200 planner's C ABI. Each test cites the
reference assertion it restates.
"""
import json
import math
import random

import pytest

from conftest import GOLDEN


def profile_text(devices, bus=True):
    """devices: dicts with id, kind, slope, intercept, [bandwidth, elem, priority,
    ops_min, ops_max, align, cache]."""
    lines = ["poas-profile v1", "", f"bus {'true' if bus else 'false'}"]
    for d in devices:
        kind = d["kind"]
        lines += ["", f"device {d['id']}", f"kind {kind}", f"slope {d['slope']!r}",
                  f"intercept {d.get('intercept', 0.0)!r}", f"bandwidth {d.get('bandwidth', 0.0)!r}",
                  f"elem_size {d.get('elem', 8)}", f"priority {d['priority']}"]
        if kind == "xpu":
            lines.append(f"align {d.get('align', 8)}")
        if kind == "cpu":
            lines.append(f"cache_bytes {d.get('cache', 33554432)}")
        lines += [f"ops_min {d.get('ops_min', 1)}", f"ops_max {d.get('ops_max', 1 << 62)}"]
    return "\n".join(lines) + "\n"


def cpu(id_, slope, intercept, prio, **kw):
    return dict(id=id_, kind="cpu", slope=slope, intercept=intercept, priority=prio, **kw)


# ------------------------------------------------------------ device model
def test_transfer_bytes_known_answer(poas):
    """proj/tests/test_device_model.cpp:80-97: 7.2e12 ops of 30000^3 at
    elem 2 -> in 2,280,000,000 B, out 480,000,000 B."""
    prof = profile_text([dict(id="x", kind="xpu", slope=1e-13, bandwidth=1e10, elem=2, priority=0)])
    assert poas.transfer_bytes(prof, "x", 7_200_000_000_000, 30000, 30000, 30000) == (
        2_280_000_000, 480_000_000)
    assert poas.transfer_bytes(prof, "x", 0, 30000, 30000, 30000) == (0, 0)
    with pytest.raises(Exception) as e:
        poas.transfer_bytes(prof, "x", 7_200_000_000_001, 30000, 30000, 30000)
    assert e.value.errc == "not_row_aligned"


def test_fit_linear_exact_and_clamp(poas):
    """proj/tests/test_device_model.cpp:44-78."""
    ops = [10**9 * i for i in range(1, 11)]
    slope, icpt = poas.fit_linear(ops, [2e-12 * o + 3e-3 for o in ops])
    assert slope == pytest.approx(2e-12, rel=1e-12) and icpt == pytest.approx(3e-3, rel=1e-12)
    secs = [2e-12 * o - 1e-3 for o in ops]  # negative intercept -> clamp
    slope, icpt = poas.fit_linear(ops, secs)
    assert icpt == 0.0
    assert slope == pytest.approx(sum(secs) / sum(ops), rel=1e-12)
    with pytest.raises(Exception) as e:
        poas.fit_linear([5, 5, 5], [1.0, 2.0, 3.0])
    assert e.value.errc == "degenerate_samples"


def test_machine_hash_topology_not_calibration(poas):
    a = profile_text([cpu("c", 1e-12, 0.0, 0), dict(id="g", kind="gpu", slope=1e-13, bandwidth=1e9,
                                                   elem=4, priority=1)])
    b = a.replace("slope 1e-13", "slope 3e-13")
    assert poas.machine_hash(a) == poas.machine_hash(b)
    assert poas.machine_hash(a) != poas.machine_hash(a.replace("bus true", "bus false"))


# ---------------------------------------------------------------- optimizer
def test_two_cpus_split_inversely_to_slopes(poas):
    """proj/tests/test_optimizer.cpp:55-76."""
    prof = profile_text([cpu("slow", 2e-12, 0.0, 1), cpu("fast", 1e-12, 0.0, 0)])
    s = poas.solve_split(prof, 30000, 10000, 10000)
    rows = {x["id"]: x["rows"] for x in s["shares"]}
    assert rows == {"slow": 10000, "fast": 20000}
    assert s["makespan"] == pytest.approx(2.0, rel=1e-12)
    assert s["lp_objective"] == pytest.approx(2.0, rel=1e-9)
    o = poas.oracle_grid_search(prof, 30000, 10000, 10000, 3000)
    assert o["makespan"] == pytest.approx(2.0, rel=1e-3)


def test_slow_device_dropped(poas):
    """proj/tests/test_optimizer.cpp:88-99."""
    prof = profile_text([cpu("fast", 1e-12, 0.0, 0), cpu("crawl", 1e-8, 0.0, 1)])
    s = poas.solve_split(prof, 60, 1000, 1000)
    assert [x["rows"] for x in s["shares"]] == [60, 0]
    assert s["makespan"] == pytest.approx(60e6 * 1e-12, rel=1e-9)


def test_single_row_goes_to_lowest_priority_number(poas):
    """proj/tests/test_optimizer.cpp:101-109."""
    prof = profile_text([cpu("a", 1e-12, 0.0, 0), cpu("b", 1e-12, 0.0, 1)])
    s = poas.solve_split(prof, 1, 5000, 5000)
    assert [x["rows"] for x in s["shares"]] == [1, 0]
    assert s["makespan"] == pytest.approx(25e6 * 1e-12, rel=1e-9)


def test_residue_goes_to_cpu_prime_m(poas, ref):
    """proj/tests/test_optimizer.cpp:111-129 (prime m = 20011)."""
    rng = random.Random(0xDEAD)
    devs = []
    for i in range(2):
        devs.append(dict(id=f"{'xpu' if i == 0 else 'gpu'}{i}", kind="xpu" if i == 0 else "gpu",
                         slope=rng.uniform(8e-14, 4e-13), intercept=rng.uniform(0.001, 0.01),
                         bandwidth=rng.uniform(16e9, 64e9), elem=rng.choice([2, 4]), priority=i,
                         align=1))
    devs.append(cpu("cpu0", 1.45e-12, 0.002, 2))
    prof = profile_text(devs)
    s = poas.solve_split(prof, 20011, 9001, 9007)
    assert sum(x["rows"] for x in s["shares"]) == 20011
    assert s["shares"][-1]["id"] == "cpu0" and s["shares"][-1]["rows"] > 0
    assert all(x["ops"] == x["rows"] * 9001 * 9007 for x in s["shares"])
    assert s == ref.solve_split(prof, 20011, 9001, 9007)


def test_lp_vs_exhaustive_gap(poas):
    """proj/tests/test_optimizer.cpp:151-166 / acceptance criterion 1: the
    planner's makespan within 0.5% of exhaustive search on random
    accelerator machines (reference random_accel_machine)."""
    rng = random.Random(0x0AC1E)
    worst = 0.0
    for _ in range(25):
        nd = rng.randint(2, 3)
        devs = []
        for i in range(nd):
            devs.append(dict(id=f"{'xpu' if i == 0 else 'gpu'}{i}", kind="xpu" if i == 0 else "gpu",
                             slope=rng.uniform(8e-14, 4e-13), intercept=rng.uniform(0.001, 0.01),
                             bandwidth=rng.uniform(16e9, 64e9), elem=rng.choice([2, 4]),
                             priority=0, align=1))
        for r, i in enumerate(sorted(range(nd), key=lambda j: devs[j]["slope"])):
            devs[i]["priority"] = r
        prof = profile_text(devs)
        m, n, k = rng.randint(20000, 60000), rng.randint(8000, 20000), rng.randint(8000, 20000)
        s = poas.solve_split(prof, m, n, k)
        o = poas.oracle_grid_search(prof, m, n, k, 400)
        worst = max(worst, (s["makespan"] - o["makespan"]) / o["makespan"])
    assert worst <= 0.005


# ------------------------------------------------------------------ adapter
def _dev(id_, kind, lo, hi, prio, **kw):
    return dict(id=id_, kind=kind, slope=1e-12, bandwidth=1e10, elem=4, priority=prio, ops_min=lo,
                ops_max=hi, align=kw.pop("align", 8), **kw)


def test_align_rows_and_unalignable_k(poas):
    """proj/tests/test_adapter.cpp:89-109 via build_tile_plan."""
    prof = profile_text([_dev("xpu0", "xpu", 1, 1 << 62, 0), _dev("gpu0", "gpu", 1, 1 << 62, 1)])
    p = poas.build_tile_plan(prof, 30000, 30000, 30000, [22330, 7670])
    assert [d["rows"] for d in p["devices"]] == [22328, 7672]  # 2 shaved rows -> gpu0
    p = poas.build_tile_plan(prof, 30000, 30000, 30000, [7, 29993])
    assert [d["rows"] for d in p["devices"]] == [0, 30000]
    with pytest.raises(Exception) as e:
        poas.build_tile_plan(prof, 30000, 30000, 30001, [16, 29984])
    assert e.value.errc == "unalignable_k"


def test_tiling_known_answers(poas):
    """proj/tests/test_adapter.cpp:147-183."""
    prof = profile_text([cpu("cpu0", 1e-12, 0.0, 0, ops_min=1_000_000_000, ops_max=8_000_000_000)])
    d = poas.build_tile_plan(prof, 2000, 2000, 2000, [2000])["devices"][0]
    assert d["k_prime"] == 2000 and d["tiles"] == [[2000, 2000, 2000]] and d["sq"] == 8e9
    d = poas.build_tile_plan(prof, 4000, 2000, 2000, [4000])["devices"][0]
    assert d["tiles"] == [[2000, 2000, 2000]] * 2 and d["sq"] == 1.6e10
    prof1 = profile_text([cpu("cpu0", 1e-12, 0.0, 0)])
    d = poas.build_tile_plan(prof1, 1, 5, 7, [1])["devices"][0]
    assert d["k_prime"] == 1 and len(d["tiles"]) == 7 and d["sq"] == 35.0


def test_window_fallback(poas):
    """proj/tests/test_adapter.cpp:216-232."""
    prof = profile_text([_dev("gpu0", "gpu", 10**9, 8 * 10**9, 0), _dev("gpu1", "gpu", 10**9, 8 * 10**9, 1)])
    p = poas.build_tile_plan(prof, 64, 100, 100, [64, 0])
    a, b = p["devices"]
    assert a["rows"] == 64 and a["window_fallback"] and a["tiles"] == [[64, 100, 100]]
    assert b["rows"] == 0 and b["tiles"] == []


def _brute_tiling(rows, k, n, lo_ops, hi_ops):
    best = None
    for kp in [d for d in range(1, k + 1) if k % d == 0]:
        for q in range(1, rows + 1):
            m_lo, m_hi, r = rows // q, -(-rows // q), rows % q
            if m_lo < 1 or any(not (lo_ops <= mm * kp * n <= hi_ops) for mm in {m_lo, m_hi}):
                continue
            sq = (k // kp) * (r * min(m_hi, kp) / max(m_hi, kp) * m_hi * kp * n +
                              (q - r) * min(m_lo, kp) / max(m_lo, kp) * m_lo * kp * n)
            cand = (sq, kp, -(k // kp) * q)
            if best is None or cand > best:
                best = cand
    return best


def test_tile_device_vs_brute_force(poas):
    """proj/tests/test_adapter.cpp:185-214 (rows, k <= 32, two windows)."""
    n = 17
    for lo, hi in ((1, 1 << 62), (3 * 17, 40 * 17)):
        prof = profile_text([_dev("d", "gpu", lo, hi, 0)])
        for rows in range(1, 33):
            for k in range(1, 33):
                brute = _brute_tiling(rows, k, n, lo, hi)
                p = poas.build_tile_plan(prof, rows, n, k, [rows])["devices"][0]
                if brute is None:
                    assert p["window_fallback"]
                    continue
                assert not p["window_fallback"]
                assert p["sq"] == pytest.approx(brute[0], rel=1e-12)
                assert p["k_prime"] == brute[1] and len(p["tiles"]) == -brute[2]


# ---------------------------------------------------------------- scheduler
def test_standalone_xpu_m16003(poas):
    """proj/tests/test_scheduler.cpp:108-136: 16003 rows on the xpu alone ->
    16000 on the xpu, 3 shaved rows on the cpu."""
    prof = (GOLDEN / "profiles" / "mach2_exact.profile").read_text()
    s = json.loads(poas.plan_standalone(prof, "xpu0", 16003, 4000, 4000))
    rows = {d["id"]: d["rows"] for d in s["devices"]}
    assert rows == {"xpu0": 16000, "gpu0": 0, "cpu0": 3}


def test_bus_exclusivity_invariant(poas):
    """proj/tests/test_scheduler.cpp:27-62: copies never overlap on the bus,
    copy-outs follow priority order, each compute follows its copy-in."""
    rng = random.Random(4)
    for name in ("mach2_exact", "mach2_seed7", "b200_like"):
        prof = (GOLDEN / "profiles" / f"{name}.profile").read_text()
        for _ in range(10):
            m = rng.randint(1000, 60000)
            s = json.loads(poas.plan(prof, m, rng.randint(1000, 30000), 8 * rng.randint(100, 3000)))
            busy = [d for d in s["devices"] if d["copy_in"][1] > d["copy_in"][0] or
                    d["copy_out"][1] > d["copy_out"][0]]
            iv = sorted([tuple(d["copy_in"]) for d in busy] + [tuple(d["copy_out"]) for d in busy])
            for (a0, a1), (b0, b1) in zip(iv, iv[1:]):
                assert b0 >= a1 - 1e-9
            for d in s["devices"]:
                assert d["compute"][0] >= d["copy_in"][1] - 1e-9
            assert s["makespan"] == max(max(d["compute"][1], d["copy_out"][1]) for d in s["devices"])


def test_table3_tops_exact():
    """acceptance.cpp:138-156: Table 3 TOps {27, 42, 52, 64, 72, 89.6}."""
    inputs = json.loads((GOLDEN / "table3.json").read_text())
    tops = [i["m"] * i["n"] * i["k"] / 1e12 for i in inputs]
    assert tops == [27.0, 42.0, 52.0, 64.0, 72.0, 89.6]


def test_format_double_roundtrip_1000(poas):
    """proj/tests/test_kv_format.cpp: %.17g reloads bit for bit (through the
    profile writer/reader)."""
    rng = random.Random(17)
    for _ in range(100):
        vals = [rng.uniform(1e-16, 1e-10) for _ in range(10)]
        prof = profile_text([dict(id=f"g{i}", kind="gpu", slope=v, intercept=v * 1e3, bandwidth=1 / v,
                                  elem=4, priority=i) for i, v in enumerate(vals)])
        canon = poas.profile_roundtrip(prof)
        assert poas.profile_roundtrip(canon) == canon
        for i, v in enumerate(vals):
            line = [ln for ln in canon.split(f"device g{i}\n")[1].splitlines() if ln.startswith("slope ")][0]
            assert float(line.split()[1]) == v


# ------------------------------------------------------------------ simplex
def test_simplex_textbook_and_failures(poas):
    """proj/tests/test_simplex.cpp:13-77."""
    # max 3x + 5y st x <= 4, 2y <= 12, 3x + 2y <= 18  ->  (2, 6), 36
    x, obj, _ = poas.solve_simplex([-3.0, -5.0], ge_a=[[-1, 0], [0, -2], [-3, -2]], ge_b=[-4, -12, -18])
    assert x == pytest.approx([2.0, 6.0]) and obj == pytest.approx(-36.0)
    x, obj, _ = poas.solve_simplex([1.0, 1.0], eq_a=[[1, 1]], eq_b=[3.0], ge_a=[[1, 0]], ge_b=[1.0])
    assert obj == pytest.approx(3.0) and x[0] >= 1 - 1e-9
    with pytest.raises(Exception) as e:  # infeasible
        poas.solve_simplex([1.0], eq_a=[[1.0]], eq_b=[1.0], ge_a=[[1.0]], ge_b=[2.0])
    assert e.value.errc == "numerical_failure"
    with pytest.raises(Exception) as e:  # unbounded
        poas.solve_simplex([-1.0], ge_a=[[1.0]], ge_b=[1.0])
    assert e.value.errc == "numerical_failure"
    # Beale's cycling example terminates under Bland's rule.
    c = [-0.75, 150.0, -0.02, 6.0]
    ge = [[-0.25, 60.0, 0.04, -9.0], [-0.5, 90.0, 0.02, -3.0], [0.0, 0.0, -1.0, 0.0]]
    x, obj, it = poas.solve_simplex(c, ge_a=ge, ge_b=[0.0, 0.0, -1.0])
    assert obj == pytest.approx(-0.05) and it < 100


def test_simplex_random_boxes(poas):
    """proj/tests/test_simplex.cpp:79-121 (box problems with known optimum)."""
    rng = random.Random(23)
    for _ in range(200):
        nv = rng.randint(1, 6)
        c = [rng.uniform(-3, 3) for _ in range(nv)]
        ub = [rng.uniform(0.5, 5) for _ in range(nv)]
        ge_a = [[-1.0 if j == i else 0.0 for j in range(nv)] for i in range(nv)]
        x, obj, _ = poas.solve_simplex(c, ge_a=ge_a, ge_b=[-u for u in ub])
        expect = sum(ci * u for ci, u in zip(c, ub) if ci < 0)
        assert obj == pytest.approx(expect, abs=1e-9)
