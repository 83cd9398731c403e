"""bench.py's reference arm on CPU (the driver runs it beside our arm): one
JSON line with the contract's keys from the reference planner + oracle port,
and silence on every rank but 0."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def run(extra_env=None, *args):
    env = dict(os.environ, **(extra_env or {}))
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", *args],
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)


def test_reference_arm_line(ref):
    r = run(None, "--size", "1024", "--steps", "1", "--warmup", "0", "--ref-rows", "64")
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "TFLOP/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["n_gpus"] == 1
    for key in ("metric", "steps", "warmup", "ms_per_step", "config", "cpu_baseline", "e2e"):
        assert key in d
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1


def test_reference_arm_other_ranks_are_silent():
    r = run({"RANK": "1", "WORLD_SIZE": "2"}, "--size", "1024", "--steps", "1", "--warmup", "0")
    assert r.returncode == 0, r.stderr
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]


def test_gpus_flag_launches_ranks_itself(ref):
    """`bench.py --gpus 2` without a launcher re-runs itself under torchrun
    with two ranks (one process per GPU); rank 0 alone prints, with
    n_gpus 2. The reference arm needs no GPU, so the
    self-launch is exercised here on CPU; the GPU arm's is in
    tests/test_gpu_multirank.py."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--size", "1024", "--steps", "1", "--warmup", "0", "--ref-rows", "64"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    assert json.loads(lines[0])["n_gpus"] == 2
