"""The library's multi-GPU path (csrc/runtime/comm.cpp + the executor's
per-repeat broadcast) on the one GPU of a test box: two processes share
cuda:0, exactly as ranks on two GPUs would run it -- shared-memory
rendezvous, CUDA IPC mappings of the upstream rank's B, copy-engine chain
with host-mapped cross-process flags, the flag-gated tensor launch and the
event-gated CUDA-core launches, alternating receive buffers over repeats --
and every rank's C is checked against the fp64 oracle. The NCCL transport
runs single-rank (NCCL refuses two ranks on one GPU).
"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
SEED = 20261017
TOL = 2e-5
PROF = "probes=4,repetitions=2,bandwidth_payload=8388608"


def _planted(profile, slope):
    out = []
    for line in profile.splitlines():
        parts = line.split()
        if len(parts) == 2 and parts[0] == "slope":
            line = f"slope {slope!r}"
        elif len(parts) == 2 and parts[0] == "intercept":
            line = "intercept 0"
        out.append(line)
    return "\n".join(out) + "\n"


def _rank_worker(rank, world, name, out_dir, m_total, n, k, panels, both_units, transport):
    sys.path.insert(0, str(ROOT))
    import torch

    import oracle
    from paper_2209_10245_b200 import poas

    torch.cuda.set_device(0)
    comm = poas.Comm(name, rank, world, 0)
    if transport == "nccl":
        comm.init_nccl()
    units = (f"gpu{rank}.tc=xpu:dev=0:sms=8:dtype=bf16:elem=2:link=hbm:probe=256-1024;"
             f"gpu{rank}.simt=gpu:dev=0:sms=4:exclusive=1:elem=4:link=hbm:probe=128-512")
    prof = poas.profile_machine(units, PROF, True)
    if both_units:  # a machine on which both units keep rows: both B paths run
        prof = _planted(prof, 2e-13)
    bw_s = comm.time_broadcast(k * n * 2, transport, 2)
    assert bw_s > 0
    bw = k * n * 2 / bw_s
    plan = poas.plan_sharded(comm.allgather(prof), [bw] * world, m_total, n, k, "reference")
    rows, row0 = plan["rows"][rank], plan["row0"][rank]
    sched = plan["plans"][rank]
    np_ = n // panels
    sa, sb = poas.stream_seed(SEED, "A"), poas.stream_seed(SEED, "B")
    dev = torch.device("cuda", 0)
    A32 = torch.empty(max(rows, 1), k, device=dev)
    A16 = torch.empty(max(rows, 1), k, device=dev, dtype=torch.bfloat16)
    poas.fill_uniform(poas.DTYPE_F32, A32.data_ptr(), k, rows, k, row0, 0, k, sa)
    poas.fill_uniform(poas.DTYPE_BF16, A16.data_ptr(), k, rows, k, row0, 0, k, sa)
    B32 = torch.zeros(panels, k, np_, device=dev)
    B16 = torch.zeros(panels, k, np_, device=dev, dtype=torch.bfloat16)
    if rank == 0:  # only the root holds B; the others must receive it
        for p in range(panels):
            poas.fill_uniform(poas.DTYPE_F32, B32[p].data_ptr(), np_, k, np_, 0, p * np_, n, sb)
            poas.fill_uniform(poas.DTYPE_BF16, B16[p].data_ptr(), np_, k, np_, 0, p * np_, n, sb)
    torch.cuda.synchronize()
    comm.register_b(B16.data_ptr(), B32.data_ptr(), k, n, panels)
    C = torch.full((max(rows, 1), n), float("nan"), device=dev)
    io = poas.GemmIO(m=rows, n=n, k=k, a_dev=A32.data_ptr(), lda_dev=k, b_dev=B32.data_ptr(), ldb_dev=np_,
                     a16_dev=A16.data_ptr(), lda16_dev=k, b16_dev=B16.data_ptr(), ldb16_dev=np_,
                     c_dev=C.data_ptr(), ldc_dev=n, resident=1, b_panels=panels, comm=comm.handle,
                     b_transport=poas.TRANSPORTS[transport])
    ex = poas.Executor(units)
    errs = []
    sd = json.loads(json.dumps(sched))
    for reps in (1, 3, 2):  # epochs 1..6: both receive buffers, twice each
        C.fill_(float("nan"))
        rep = ex.execute(json.dumps(sched), io, reps)
        torch.cuda.synchronize()
        A = oracle.fill_uniform(rows, k, sa, row0, 0, k)
        exp = oracle.expected_c(sd, A, oracle.fill_uniform(k, n, sb),
                                {f"gpu{rank}.tc": 2, f"gpu{rank}.simt": 0})
        errs.append(oracle.rel_frobenius(C[:rows].cpu().numpy(), exp))
        assert rep["repeats"] == reps
    comm.barrier()
    Path(out_dir, f"r{rank}.json").write_text(json.dumps({
        "rows": plan["rows"], "errs": errs, "bw": bw,
        "unit_rows": {d["id"]: d["rows"] for d in sd["devices"]}}))
    del ex
    comm.close()


def _run(tmp_path, world, transport="ce", both_units=False, m_total=1536, n=2048, k=512, panels=4):
    import torch.multiprocessing as mp

    name = f"g{os.getpid()}_{world}_{transport}_{int(both_units)}"
    mp.start_processes(_rank_worker, args=(world, name, str(tmp_path), m_total, n, k, panels, both_units,
                                           transport),
                       nprocs=world, join=True, start_method="spawn")
    return [json.loads((tmp_path / f"r{r}.json").read_text()) for r in range(world)]


@pytest.fixture(scope="module")
def gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


@pytest.mark.timeout(600)
def test_two_ranks_copy_engine_chain(gpu, tmp_path):
    """Two ranks: rank 1 receives B only through the chain; C exact on both
    ranks for 6 consecutive broadcasts (both receive buffers)."""
    res = _run(tmp_path, 2)
    assert sum(res[0]["rows"]) == 1536
    for r in res:
        assert max(r["errs"]) <= TOL, r
        assert r["bw"] > 0


@pytest.mark.timeout(600)
def test_three_ranks_both_units_read_broadcast_b(gpu, tmp_path):
    """Three ranks (two chain hops), both units busy: the tensor unit's one
    flag-gated launch reads the 16-bit B, the CUDA-core unit's per-panel
    launches read the fp32 B behind the per-panel events."""
    res = _run(tmp_path, 3, both_units=True, m_total=2304)
    for r in res:
        assert max(r["errs"]) <= TOL, r
    assert all(v > 0 for v in res[2]["unit_rows"].values()), res[2]["unit_rows"]


@pytest.mark.timeout(600)
def test_single_rank_nccl_transport(gpu, tmp_path):
    """The NCCL transport through the same executor path (one rank)."""
    res = _run(tmp_path, 1, transport="nccl")
    assert max(res[0]["errs"]) <= TOL
