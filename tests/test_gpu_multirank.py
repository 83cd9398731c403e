"""The multi-rank bench path on the one GPU of a test box: `bench.py --gpus
2` launches its own two ranks (no external launcher), both on cuda:0 --
level-1 rows from the C++ two-level planner over both ranks' profiles, B
broadcast from rank 0 by the library inside every executor step (copy-
engine chain over CUDA IPC), max-over-ranks timing, per-rank C checks, the
C4 strong-scaling measurement, e2e. The measured N > 1 configuration is one
GPU per rank; this checks the orchestration and every rank's C, not speed."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _env():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    env["OMP_NUM_THREADS"] = "2"
    return env


def test_two_ranks_one_gpu_bench(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--size=2048", "--steps", "3", "--warmup", "3",
           "--no-cpu-baseline", "--no-e2e-cpu", "--c4-steps", "2", "--save", str(tmp_path / "out")]
    r = subprocess.run(cmd, cwd=ROOT, env=_env(), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0
    cfg = line["config"]
    assert cfg["m"] == 2 * 2048 and sum(cfg["level1_rows_per_gpu"]) == 4096
    assert len(cfg["level1_rows_per_gpu"]) == 2 and min(cfg["level1_rows_per_gpu"]) > 0
    assert cfg["b_transport"].startswith("ce") and cfg["level1_link_gbs"] > 0
    assert cfg["c_check"]["max_rel_err"] <= cfg["c_check"]["tol"]
    assert cfg["c_check"]["sampled_rows"]["rel_frobenius"] <= cfg["c_check"]["tol"]
    c4 = cfg["c4"]
    assert c4["scaling"] == "strong" and sum(c4["level1_rows_per_gpu"]) == 65536 and c4["value"] > 0
    assert c4["c_check"]["sampled_rows"]["rel_frobenius"] <= c4["c_check"]["tol"]
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert e2e["synchronous"]["value"] > 0 and ("single_step" in e2e or "pipelined" in e2e)


def test_two_ranks_strong_scaling_c4_shape_torchrun(tmp_path):
    """Config C4's shape (M_total rows split over the ranks, N = K), small,
    launched the way the driver does (torchrun)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", str(ROOT / "bench.py"), "--gpus", "2",
           "--m-total=6144", "--size=2048", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
           "--no-e2e"]
    r = subprocess.run(cmd, cwd=ROOT, env=_env(), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    cfg = line["config"]
    assert line["scaling"] == "strong" and cfg["m"] == 6144 and sum(cfg["level1_rows_per_gpu"]) == 6144
    assert cfg["c_check"]["max_rel_err"] <= cfg["c_check"]["tol"]
