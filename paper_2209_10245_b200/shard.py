"""Multi-GPU POAS: two-level planning and the sharded step.

Level 1 splits the rows of A across the G GPUs of a box with the *same*
planner: every GPU is one device of kind xpu whose model is its units'
combined throughput, on private links (``bus false`` -- NVSwitch gives every
GPU its own full-bandwidth port, the reference's private-link timeline,
proj/src/timeline.cpp:24-35). For identical GPUs the reference LP splits
exactly evenly. Level 2 is each rank's ordinary per-GPU plan over its own
units. The only exchange in the data path is B: resident on rank 0 and
broadcast (NCCL over NVLink on GPUs, gloo in the CPU tests) once per GEMM.
"""
from __future__ import annotations

import json
import math
from typing import Sequence

from . import poas


def _parse_devices(profile: str) -> list[dict]:
    devs, cur = [], None
    for line in profile.splitlines():
        if line.startswith("device "):
            cur = {"id": line.split(" ", 1)[1]}
            devs.append(cur)
        elif cur is not None and " " in line:
            key, val = line.split(" ", 1)
            cur[key] = val
    return devs


def level1_profile(world: int, per_gpu_profile: str, link_bandwidth: float) -> str:
    """G identical "gpu<r>" devices, each the aggregate of one GPU's units:
    slope = 1 / sum(1/slope_u) (throughputs add), intercept = max, elem 2,
    align = lcm of the units' aligns, private links."""
    devs = [d for d in _parse_devices(per_gpu_profile) if d["kind"] != "cpu"]
    if not devs:
        raise ValueError("per-GPU profile has no GPU units")
    slope = 1.0 / sum(1.0 / float(d["slope"]) for d in devs)
    intercept = max(float(d["intercept"]) for d in devs)
    align = 1
    for d in devs:
        if d["kind"] == "xpu":
            align = align * int(d["align"]) // math.gcd(align, int(d["align"]))
    lines = ["poas-profile v1", "", "bus false"]
    for r in range(world):
        lines += ["", f"device gpu{r}", "kind xpu", f"slope {slope!r}", f"intercept {intercept!r}",
                  f"bandwidth {float(link_bandwidth)!r}", "elem_size 2", f"priority {r}",
                  f"align {align}", "ops_min 1", f"ops_max {1 << 62}"]
    return "\n".join(lines) + "\n"


def shard_rows(world: int, m: int, n: int, k: int, per_gpu_profile: str,
               link_bandwidth: float = 7.7e11) -> list[int]:
    """Rows of A per rank from the level-1 plan (schedule order = rank order)."""
    sched = json.loads(poas.plan(level1_profile(world, per_gpu_profile, link_bandwidth), m, n, k))
    rows = {d["id"]: d["rows"] for d in sched["devices"]}
    return [rows[f"gpu{r}"] for r in range(world)]


def row_offsets(rows: Sequence[int]) -> list[int]:
    out, at = [], 0
    for r in rows:
        out.append(at)
        at += r
    return out


def broadcast_b(tensors, src: int = 0, group=None) -> None:
    """The one data-path collective: B (every precision a unit consumes)
    from the rank that holds it to all others."""
    import torch.distributed as dist

    for t in tensors:
        dist.broadcast(t, src=src, group=group)


def sharded_step(executor: "poas.Executor", schedule: str, io: "poas.GemmIO", b_tensors,
                 repeats: int = 1, group=None) -> dict:
    """One co-executed GEMM on this rank's shard: receive B, run the plan."""
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_world_size(group) > 1:
        broadcast_b(b_tensors, 0, group)
    return executor.execute(schedule, io, repeats)
