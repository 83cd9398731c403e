"""The multi-rank bench path (N > 1: level-1 row shards, B broadcast from
rank 0 in column panels with per-panel readiness events, max-over-ranks
timing, per-rank C check) run end to end on the one GPU of a test box: two
ranks share cuda:0 over gloo (POAS_DIST_BACKEND=gloo). The measured N > 1
configuration is NCCL with one GPU per rank; this checks the orchestration
and every rank's C, not the speed."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_two_ranks_one_gpu_bench(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, POAS_DIST_BACKEND="gloo", OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29531", str(ROOT / "bench.py"), "--gpus", "2",
           "--size=2048", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e-cpu",
           "--save", str(tmp_path / "out")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0
    cfg = line["config"]
    assert cfg["m"] == 2 * 2048 and cfg["level1_rows_per_gpu"] == [2048, 2048]
    assert cfg["dist_backend"] == "gloo"
    assert cfg["c_check"]["max_rel_err"] <= cfg["c_check"]["tol"]
    e2e = line["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert e2e["synchronous"]["value"] > 0 and ("single_step" in e2e or "pipelined" in e2e)


def test_two_ranks_strong_scaling_c4_shape(tmp_path):
    """Config C4's shape (M_total rows split over the ranks, N = K), small."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, POAS_DIST_BACKEND="gloo", OMP_NUM_THREADS="2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", str(ROOT / "bench.py"), "--gpus", "2",
           "--m-total=6144", "--size=2048", "--steps", "3", "--warmup", "3", "--no-cpu-baseline",
           "--no-e2e"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    cfg = line["config"]
    assert line["scaling"] == "strong" and cfg["m"] == 6144 and cfg["level1_rows_per_gpu"] == [3072, 3072]
    assert cfg["c_check"]["max_rel_err"] <= cfg["c_check"]["tol"]
