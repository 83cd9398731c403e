"""Multi-GPU POAS: the two-level plan and the job's communicator.

Thin bindings over the C ABI (include/poas_b200.h "Multi-GPU"):
  * poas_b200_plan_sharded -- level 1 splits the rows of A across the GPUs
    of a box with the same planner, every GPU one xpu device whose model is
    its units' combined throughput on a private link (bus false, the
    reference's NVSwitch-shaped timeline, proj/src/timeline.cpp:24-35) whose
    bandwidth is the measured B broadcast; level 2 is each GPU's own plan of
    its rows (csrc/planner/sharded.cpp);
  * poas_b200_comm_* -- one process per GPU joined through shared memory; the
    executor broadcasts B itself (copy-engine chain over CUDA IPC, or NCCL).
"""
from __future__ import annotations

import os
from typing import Sequence

from . import poas


def plan(gpu_profiles: Sequence[str], link_bandwidth: Sequence[float], m: int, n: int, k: int,
         policy: str = "reference") -> dict:
    """{"level1_profile", "level1", "rows", "row0", "plans"} (poas_b200_plan_sharded)."""
    return poas.plan_sharded(gpu_profiles, link_bandwidth, m, n, k, policy)


def shard_rows(world: int, m: int, n: int, k: int, per_gpu_profile: str,
               link_bandwidth: float = 7.7e11) -> list[int]:
    """Rows of A per rank for `world` identical GPUs (rank order)."""
    return plan([per_gpu_profile] * world, [link_bandwidth] * world, m, n, k)["rows"]


def row_offsets(rows: Sequence[int]) -> list[int]:
    out, at = [], 0
    for r in rows:
        out.append(at)
        at += r
    return out


def comm_name() -> str:
    """A rendezvous token identical on every rank of one launch and unique
    per launch: the launcher's pid (the ranks' common parent), run id and
    port (torchrun exports both)."""
    run = os.environ.get("TORCHELASTIC_RUN_ID", "none")
    port = os.environ.get("MASTER_PORT", "0")
    tok = "".join(ch if ch.isalnum() else "_" for ch in f"{os.getppid()}_{run}_{port}")
    return f"job_{tok}"
