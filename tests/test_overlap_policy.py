"""The "overlap" planner policy (B200 extension; paper PAPER.md:486-489:
"could be improved using CUDA streams and overlapping the computation with
memory copies ... the performance predictor can be adapted to predict the
memory copies with or without overlap").

The C++ planner's overlapped timeline is checked against an independent
restatement here (`overlap_timeline`), on hand-computed and random machines;
the row parts, the subset/part choice, the schedule interchange format and
the untouched reference policy are checked too.
"""
import json
import random

import pytest

from conftest import GOLDEN
from test_planner_parity import random_dims, random_profile

REL = 1e-9


def parse_profile(text):
    devs, cur, bus = [], None, True
    for line in text.splitlines():
        p = line.split()
        if len(p) != 2:
            continue
        if p[0] == "bus":
            bus = p[1] == "true"
        elif p[0] == "device":
            cur = {"id": p[1]}
            devs.append(cur)
        elif cur is not None:
            cur[p[0]] = p[1]
    for d in devs:
        for key in ("slope", "intercept", "bandwidth"):
            d[key] = float(d[key])
        d["elem_size"] = int(d["elem_size"])
        d["priority"] = int(d["priority"])
    return devs, bus


def split(extent, parts, block):
    """poas::overlap_split: whole blocks spread evenly, tail on the last."""
    if extent <= 0:
        return []
    blocks = extent // block
    if blocks == 0:
        return [extent]
    q = max(1, min(parts, blocks))
    out = [(blocks // q + (1 if p < blocks % q else 0)) * block for p in range(q)]
    out[-1] += extent % block
    return out


def row_parts(rows, parts):
    return split(rows, parts, 256)


def link_order(R, Q):
    """poas::overlap_link_order: A while proportionally behind."""
    out, a, b = [], 0, 0
    while a < R or b < Q:
        if b >= Q or (a < R and a * Q <= b * R):
            out.append(("A", a))
            a += 1
        else:
            out.append(("B", b))
            b += 1
    return out


def block_order(R, Q):
    """poas::overlap_block_order: (part, panel, ready item) as items land."""
    out, a, b = [], 0, 0
    for k, (kind, _) in enumerate(link_order(R, Q)):
        if kind == "A":
            out += [(a, j, k) for j in range(b)]
            a += 1
        else:
            out += [(i, b, k) for i in range(a)]
            b += 1
    return out


def overlap_timeline(devs, bus, grids, m, n, k):
    """Restatement of poas::evaluate_overlap_timeline over each unit's grid
    of row parts x column panels: link items (A parts, B panels) back to
    back on the host->device queue in link order; block b computes after its
    ready item and block b-1; its C (fp32) leaves after that and after the
    previous copy-out on the device->host queue; queues shared in priority
    order when `bus`. Returns ({id: (copy_in, compute, copy_out)}, makespan)."""
    h2d = d2h = 0.0
    out, makespan = {}, 0.0
    for d in sorted(devs, key=lambda x: x["priority"]):
        rp, cp = grids[d["id"]]
        slope, icpt = d["slope"], d["intercept"]
        if d["kind"] == "cpu":
            c = sum(slope * r * n * k + icpt for r in rp)
            out[d["id"]] = ((0.0, 0.0), (0.0, c), (c, c))
            makespan = max(makespan, c)
            continue
        if not rp:
            at = h2d if bus else 0.0
            out[d["id"]] = ((at, at), (at, at), (at, at))
            continue
        bw, e = d["bandwidth"], d["elem_size"]
        t_in = h2d if bus else 0.0
        start_in = t_in
        landed = []
        for kind, x in link_order(len(rp), len(cp)):
            t_in += e * k * (rp[x] if kind == "A" else cp[x]) / bw
            landed.append(t_in)
        free_out = d2h if bus else 0.0
        c_end, c_start, o_start = 0.0, None, None
        for i, j, ready in block_order(len(rp), len(cp)):
            cs = max(landed[ready], c_end)
            c_end = cs + slope * rp[i] * cp[j] * k + icpt
            os_ = max(c_end, free_out)
            free_out = os_ + 4.0 * rp[i] * cp[j] / bw + (20e-6 if len(rp) * len(cp) > 1 else 0.0)
            if c_start is None:
                c_start, o_start = cs, os_
        out[d["id"]] = ((start_in, t_in), (c_start, c_end), (o_start, free_out))
        if bus:
            h2d, d2h = t_in, free_out
        makespan = max(makespan, free_out)
    return out, makespan


def grid_of(tiles, n):
    """Row parts and column panels of an overlap schedule's part-major tiles."""
    cp, covered = [], 0
    for t in tiles:
        if covered >= n:
            break
        cp.append(t["n"])
        covered += t["n"]
    q = len(cp)
    rp = [tiles[p * q]["m"] for p in range(len(tiles) // q)] if q else []
    return rp, cp


def check_against_restatement(poas, prof, m, n, k):
    s = json.loads(poas.plan_policy(prof, m, n, k, "overlap"))
    devs, bus = parse_profile(prof)
    grids = {}
    for d in s["devices"]:
        dev = next(x for x in devs if x["id"] == d["id"])
        if dev["kind"] == "cpu":
            grids[d["id"]] = ([d["rows"]] if d["rows"] else [], [n])
        elif d["rows"] == 0:
            assert d["tiles"] == []
            grids[d["id"]] = ([], [])
        else:
            # link units: an R x Q grid of full-K blocks, part-major
            assert all(t["k"] == k for t in d["tiles"])
            rp, cp = grid_of(d["tiles"], n)
            assert len(rp) * len(cp) == len(d["tiles"])
            assert [t["m"] for t in d["tiles"]] == [r for r in rp for _ in cp]
            assert [t["n"] for t in d["tiles"]] == cp * len(rp)
            assert sum(rp) == d["rows"] and sum(cp) == n
            assert rp == row_parts(d["rows"], len(rp)) and cp == split(n, len(cp), 256)
            grids[d["id"]] = (rp, cp)
    tl, makespan = overlap_timeline(devs, bus, grids, m, n, k)
    assert s["makespan"] == pytest.approx(makespan, rel=REL, abs=2e-9)
    for d in s["devices"]:
        want = tl[d["id"]]
        for key, iv in zip(("copy_in", "compute", "copy_out"), want):
            # schedule times are %.9f (reference proj/src/scheduler.cpp:96-100)
            assert d[key][0] == pytest.approx(iv[0], abs=1e-9), (d["id"], key)
            assert d[key][1] == pytest.approx(iv[1], abs=1e-9), (d["id"], key)
    return s


def test_link_and_block_order():
    assert link_order(3, 1) == [("A", 0), ("B", 0), ("A", 1), ("A", 2)]
    assert link_order(2, 2) == [("A", 0), ("B", 0), ("A", 1), ("B", 1)]
    assert link_order(1, 3) == [("A", 0), ("B", 0), ("B", 1), ("B", 2)]
    assert block_order(2, 2) == [(0, 0, 1), (1, 0, 2), (0, 1, 3), (1, 1, 3)]
    for R, Q in ((1, 1), (4, 2), (3, 5), (8, 8)):
        blocks = block_order(R, Q)
        assert sorted((i, j) for i, j, _ in blocks) == [(i, j) for i in range(R) for j in range(Q)]


def test_row_parts():
    assert row_parts(16384, 64) == [256] * 64
    assert row_parts(1000, 4) == [256, 256, 488]
    assert row_parts(100, 8) == [100]
    assert row_parts(600, 8) == [256, 344]


def test_overlap_b200_e2e_profile(poas):
    """The e2e machine of the r1i box (bf16 link for the tensor unit): the
    overlapped plan keeps the tensor unit alone, cuts it into row parts and
    predicts B + the C stream instead of copy-in + compute + copy-out."""
    prof = (GOLDEN / "profiles" / "b200_e2e_r1i.profile").read_text()
    m = n = k = 16384
    seq = json.loads(poas.plan_policy(prof, m, n, k, "best-subset"))
    s = check_against_restatement(poas, prof, m, n, k)
    rows = {d["id"]: d["rows"] for d in s["devices"]}
    assert rows == {"gpu0.tc": 16384, "cpu0": 0, "gpu0.simt": 0}
    tc = next(d for d in s["devices"] if d["id"] == "gpu0.tc")
    rp, cp = grid_of(tc["tiles"], n)
    assert len(rp) >= 4 and len(cp) >= 2, (len(rp), len(cp))  # a 2-D grid wins here
    # copies overlap compute: C leaves while A and B are still arriving
    assert tc["copy_out"][0] < tc["copy_in"][1]
    # floor: the busier link direction (host->device: A and B, 2 bytes; C
    # back is 4 bytes, as much) -- the 1-D scheme (B, then A parts) pays
    # all of B before any C can leave
    devs, _ = parse_profile(prof)
    bw = next(d for d in devs if d["id"] == "gpu0.tc")["bandwidth"]
    floor = max(2 * (m * k + k * n), 4 * m * n) / bw
    one_d = (2 * k * n + 4 * m * n) / bw
    assert floor < s["makespan"] < 0.95 * one_d
    # the synchronous plan charges the 2-byte unit's C at 2 bytes (reference
    # transfer_bytes), yet overlap still predicts less
    assert s["makespan"] < seq["makespan"]
    assert poas.schedule_roundtrip(json.dumps(s)) == poas.plan_policy(prof, m, n, k, "overlap")


def test_overlap_hand_computed(poas):
    """One link unit, exact numbers: bw 1e9 B/s, e=4, slope 1e-12, no
    intercept, 1024x512x256. Whatever grid the policy picks, its makespan
    is the pipeline recurrence over that grid written out by hand here, and
    beats the synchronous copy-in, compute, copy-out."""
    prof = "\n".join([
        "poas-profile v1", "", "bus true", "",
        "device g", "kind gpu", "slope 1e-12", "intercept 0", "bandwidth 1000000000",
        "elem_size 4", "priority 0", "ops_min 1", "ops_max 1000000000000", ""])
    m, n, k = 1024, 512, 256
    s = check_against_restatement(poas, prof, m, n, k)
    rp, cp = grid_of(s["devices"][0]["tiles"], n)
    # hand-rolled: items in link order, blocks as they become computable
    landed, t = {}, 0.0
    for kind, x in link_order(len(rp), len(cp)):
        t += 4 * k * (rp[x] if kind == "A" else cp[x]) / 1e9
        landed[(kind, x)] = t
    c_end = o_end = 0.0
    for i, j, _ in block_order(len(rp), len(cp)):
        c_end = max(landed[("A", i)], landed[("B", j)], c_end) + 1e-12 * rp[i] * cp[j] * k
        o_end = max(c_end, o_end) + 4 * rp[i] * cp[j] / 1e9 + (20e-6 if len(rp) * len(cp) > 1 else 0.0)
    assert s["makespan"] == pytest.approx(o_end, abs=2e-9)
    seq = 4 * (m * k + k * n) / 1e9 + 1e-12 * m * n * k + 4 * m * n / 1e9
    assert s["makespan"] < seq


def test_overlap_random_machines(poas):
    rng = random.Random(7)
    checked = 0
    for _ in range(120):
        nd = rng.randint(1, 4)
        prof = random_profile(rng, nd, with_cpu=rng.random() < 0.5, bus=rng.random() < 0.7)
        m, n, k = random_dims(rng)
        try:
            ref = json.loads(poas.plan_policy(prof, m, n, k, "best-subset"))
        except Exception:
            continue
        s = check_against_restatement(poas, prof, m, n, k)
        assert sum(d["rows"] for d in s["devices"]) == m
        assert s["machine_hash"] == ref["machine_hash"]
        checked += 1
    assert checked > 60


def test_reference_policy_unchanged_by_overlap(poas, ref):
    prof = (GOLDEN / "profiles" / "b200_like.profile").read_text()
    assert poas.plan_policy(prof, 16384, 16384, 16384, "reference") == ref.plan(prof, 16384, 16384, 16384)
    from paper_2209_10245_b200 import PoasError

    with pytest.raises(PoasError):
        poas.plan_policy(prof, 16384, 16384, 16384, "no-such-policy")


def _overlap_report(s, finish_scale, compute_scale=1.0):
    devs = []
    for d in s["devices"]:
        ci = d["copy_in"][1] - d["copy_in"][0]
        cc = d["compute"][1] - d["compute"][0]
        co = d["copy_out"][1] - d["copy_out"][0]
        fin = d["copy_out"][1]

        def ph(pred, f):
            return {"measured": pred * f, "predicted": pred, "error_pct": 0.0}

        devs.append({"id": d["id"], "rows": d["rows"], "copy_in": ph(ci, 1.0), "compute": ph(cc, compute_scale),
                     "copy_out": ph(co, 1.0), "finish": ph(fin, finish_scale), "overlapped": d["rows"] > 0})
    return {"measured_makespan": s["makespan"] * finish_scale, "predicted_makespan": s["makespan"],
            "makespan_error_pct": 0.0, "devices": devs}


def test_refit_of_overlapped_runs(poas):
    """Dynamic re-fit of an overlapped run (csrc/planner/dynamic.cpp): a
    link-bound unit's finish ratio rescales its link bandwidth (the copy
    spans overlap and the directions contend, so their sum is no measure);
    its compute model is left alone. Re-planned, the prediction follows."""
    prof = (GOLDEN / "profiles" / "b200_e2e_r1i.profile").read_text()
    m = n = k = 16384
    s = json.loads(poas.plan_policy(prof, m, n, k, "overlap"))
    rep = _overlap_report(s, finish_scale=1.08, compute_scale=1.3)
    out = poas.refit_profile(prof, rep, 1.0)
    before, _ = parse_profile(prof)
    after, _ = parse_profile(out)
    b = {d["id"]: d for d in before}
    a = {d["id"]: d for d in after}
    assert a["gpu0.tc"]["bandwidth"] == pytest.approx(b["gpu0.tc"]["bandwidth"] / 1.08, rel=1e-12)
    assert a["gpu0.tc"]["slope"] == b["gpu0.tc"]["slope"]
    s2 = json.loads(poas.plan_policy(out, m, n, k, "overlap"))
    assert s2["makespan"] == pytest.approx(s["makespan"] * 1.08, rel=0.01)
    # without the flag the same numbers are a synchronous run: compute moves
    for d in rep["devices"]:
        d.pop("overlapped")
    out2 = poas.refit_profile(prof, rep, 1.0)
    a2 = {d["id"]: d for d in parse_profile(out2)[0]}
    assert a2["gpu0.tc"]["slope"] == pytest.approx(b["gpu0.tc"]["slope"] * 1.3, rel=1e-12)
