"""N > 1 host logic on CPU: world_size-2 gloo processes run the sharded
POAS step end to end with CPU units (the executor's host path), B broadcast
from rank 0, and the gathered C checked against the fp64 oracle. Also the
level-1 (per-GPU) split of BASELINE config C4 across 2/4/8 GPUs."""
import json
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2209_10245_b200 import poas, shard

    # file rendezvous: no port races between concurrently running suites
    dist.init_process_group("gloo", init_method=f"file://{out_dir}/rdzv", rank=rank,
                            world_size=world)
    m_total, n, k = 520, 192, 160
    units = f"cpu{rank}=cpu:threads=2"
    # a fixed profile (the probes are not under test here; two ranks timing
    # tiny probes on a shared CPU could fit a degenerate slope)
    prof = (f"poas-profile v1\n\nbus true\n\ndevice cpu{rank}\nkind cpu\nslope 2e-10\n"
            "intercept 0.0001\nbandwidth 0\nelem_size 4\npriority 0\ncache_bytes 33554432\n"
            "ops_min 110592\nops_max 2097152\n")
    prof = poas.profile_roundtrip(prof)
    # level-1 split: planned on rank 0, shared (every rank could plan it too:
    # the planner is deterministic given the profile)
    obj = [None]
    if rank == 0:
        gpu_like = prof.replace("kind cpu", "kind gpu").replace("cache_bytes", "bandwidth_x")
        gpu_like = "\n".join(l for l in gpu_like.splitlines() if not l.startswith("bandwidth_x"))
        gpu_like = gpu_like.replace("bandwidth 0", "bandwidth 1e11")
        obj = [shard.shard_rows(world, m_total, n, k, gpu_like, 1e11)]
    dist.broadcast_object_list(obj, src=0)
    rows = obj[0]
    r0 = shard.row_offsets(rows)[rank]
    m = rows[rank]
    sched = poas.plan(prof, m, n, k)
    assert sched == oracle.ref.plan(prof, m, n, k)

    sa, sb = poas.stream_seed(20261017, "A"), poas.stream_seed(20261017, "B")
    A = oracle.fill_uniform(m, k, sa, row0=r0, total_cols=k)  # this rank's rows only
    B = torch.zeros(k, n) if rank else torch.from_numpy(oracle.fill_uniform(k, n, sb))
    C = np.full((m, n), np.nan, dtype=np.float32)
    io = poas.GemmIO(m=m, n=n, k=k, a_host=A.ctypes.data, lda_host=k, b_host=B.data_ptr(),
                     ldb_host=n, c_host=C.ctypes.data, ldc_host=n, resident=1)
    ex = poas.Executor(units)
    # B to every rank (host-CPU units read host B; the GPU path's broadcast
    # is the library's, tests/test_gpu_multirank.py)
    dist.broadcast(B, src=0)
    rep = ex.execute(sched, io, 1)
    assert rep["devices"][0]["rows"] == m
    gathered = [None] * world
    dist.all_gather_object(gathered, (r0, C))
    if rank == 0:
        full = np.concatenate([c for _, c in sorted(gathered, key=lambda t: t[0])])
        Afull = oracle.fill_uniform(m_total, k, sa)
        ref = oracle.gemm_rows_f64(Afull, oracle.fill_uniform(k, n, sb), 0)
        err = oracle.rel_frobenius(full, ref)
        Path(out_dir, "result.json").write_text(json.dumps({"rows": rows, "err": err}))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_gemm(tmp_path, ref):
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    res = json.loads((tmp_path / "result.json").read_text())
    assert sum(res["rows"]) == 520 and len(res["rows"]) == 2
    assert res["err"] <= 2e-5


@pytest.mark.parametrize("world", [2, 4, 8])
def test_level1_split_config_c4(poas, world):
    """C4: 65536 x 8192 x 8192 over G identical B200s -> equal shards (SURVEY
    Appendix B: 32768x2 / 16384x4 / 8192x8)."""
    from paper_2209_10245_b200 import shard

    per_gpu = ("poas-profile v1\n\nbus true\n\ndevice gpu0.tc\nkind xpu\nslope 1.45e-15\n"
               "intercept 2.0000000000000002e-05\nbandwidth 6500000000000\nelem_size 2\npriority 0\n"
               "align 8\nops_min 549755813888\nops_max 4398046511104\n\ndevice gpu0.simt\nkind gpu\n"
               "slope 3.5e-14\nintercept 2.0000000000000002e-05\nbandwidth 6500000000000\n"
               "elem_size 4\npriority 1\nops_min 134217728\nops_max 8589934592\n")
    rows = shard.shard_rows(world, 65536, 8192, 8192, per_gpu, 9e11)
    assert rows == [65536 // world] * world


def _level1_restated(world, per_gpu_profile, link_bandwidth):
    """The round-1 Python restatement of the level-1 profile (aggregate
    slope = 1/sum(1/slope_u), intercept = max, align = lcm over xpu units,
    private links; tile window from 2^40 MACs, see csrc/planner/sharded.cpp)
    -- the C++ planner must produce the same plan."""
    import math

    devs, cur = [], None
    for line in per_gpu_profile.splitlines():
        if line.startswith("device "):
            cur = {"id": line.split(" ", 1)[1]}
            devs.append(cur)
        elif cur is not None and " " in line:
            key, val = line.split(" ", 1)
            cur[key] = val
    devs = [d for d in devs if d["kind"] != "cpu"]
    inv = 0.0  # left-to-right (Python 3.12's sum() compensates; the C++ does not)
    for d in devs:
        inv += 1.0 / float(d["slope"])
    slope = 1.0 / inv
    intercept = max(float(d["intercept"]) for d in devs)
    align = 1
    for d in devs:
        if d["kind"] == "xpu":
            align = align * int(d["align"]) // math.gcd(align, int(d["align"]))
    lines = ["poas-profile v1", "", "bus false"]
    for r in range(world):
        lines += ["", f"device gpu{r}", "kind xpu", f"slope {slope!r}", f"intercept {intercept!r}",
                  f"bandwidth {float(link_bandwidth)!r}", "elem_size 2", f"priority {r}",
                  f"align {align}", f"ops_min {1 << 40}", f"ops_max {1 << 62}"]
    return "\n".join(lines) + "\n"


def test_level1_plan_matches_round1_restatement(poas, ref):
    """The C++ two-level planner's level 1 == the round-1 Python level-1
    profile planned by the reference planner, on random per-GPU profiles
    and shapes; level 2 == the reference plan of each GPU's rows."""
    import random

    from paper_2209_10245_b200 import shard
    from test_planner_parity import random_dims, random_profile

    rng = random.Random(11)
    checked = 0
    for _ in range(300):
        world = rng.choice([1, 2, 3, 4, 8])
        prof = poas.profile_roundtrip(random_profile(rng, rng.randint(1, 3), rng.random() < 0.3, True))
        if all("kind cpu" in blk for blk in prof.split("\n\n")[2:]):
            continue
        m, n, k = random_dims(rng)
        bw = rng.choice([9e11, 4.5e11, 7.7e11])
        l1 = _level1_restated(world, prof, bw)
        try:
            want = json.loads(ref.plan(l1, m, n, k))
        except Exception:
            with pytest.raises(Exception):
                shard.plan([prof] * world, [bw] * world, m, n, k)
            continue
        got = shard.plan([prof] * world, [bw] * world, m, n, k)
        assert got["level1"] == want, (world, m, n, k)
        assert poas.profile_roundtrip(got["level1_profile"]) == poas.profile_roundtrip(l1)
        assert got["rows"] == [d["rows"] for d in want["devices"]]
        for g, r in enumerate(got["rows"]):
            if r:
                assert got["plans"][g] == json.loads(ref.plan(prof, r, n, k))
            else:
                assert got["plans"][g] is None
        checked += 1
    assert checked >= 150


def test_level1_heterogeneous_gpus(poas):
    """A GPU whose units are half as fast gets fewer rows (not quite half:
    both pay the same B transfer and per-row A transfer on their links): the
    level-1 plan reacts to a slower (throttled) GPU, and the two finish
    together in its timeline."""
    from paper_2209_10245_b200 import shard

    def gpu(slope):
        return poas.profile_roundtrip(
            "poas-profile v1\n\nbus true\n\ndevice tc\nkind xpu\n"
            f"slope {slope!r}\nintercept 2e-05\nbandwidth 6.5e12\nelem_size 2\npriority 0\nalign 1\n"
            "ops_min 549755813888\nops_max 4398046511104\n")

    p = shard.plan([gpu(7e-16), gpu(1.4e-15)], [9e11, 9e11], 65536, 8192, 8192)
    fast, slow = p["rows"]
    assert fast + slow == 65536 and p["row0"] == [0, fast]
    assert 1.4 < fast / slow < 2.0, p["rows"]
    fin = [d["copy_out"][1] for d in p["level1"]["devices"]]
    assert abs(fin[0] - fin[1]) / max(fin) < 0.01, fin


def _comm_worker(rank, world, name, out_dir):
    sys.path.insert(0, str(ROOT))
    from paper_2209_10245_b200 import poas

    c = poas.Comm(name, rank, world, -1)
    got = c.allgather(f"rank {rank} says \"hi\"\n" * (rank + 1))
    mx = c.max(float(rank * 10))
    c.barrier()
    Path(out_dir, f"r{rank}.json").write_text(json.dumps({"all": got, "max": mx}))
    c.close()


@pytest.mark.parametrize("world", [2, 3])
def test_host_comm_allgather_barrier(tmp_path, world):
    """The library communicator's host side (shared-memory rendezvous,
    barrier, all-gather, max) across real processes."""
    name = f"t{os.getpid()}_{world}"
    mp.start_processes(_comm_worker, args=(world, name, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        res = json.loads((tmp_path / f"r{r}.json").read_text())
        assert res["all"] == [f"rank {q} says \"hi\"\n" * (q + 1) for q in range(world)]
        assert res["max"] == 10.0 * (world - 1)
