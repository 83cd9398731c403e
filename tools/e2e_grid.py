"""Pipelined e2e step time vs the overlap grid (dev tool).

    python tools/e2e_grid.py

Plans the 16384^3 e2e GEMM with the overlap policy (bf16 host A/B, fp32 C,
the tensor unit over PCIe), then rewrites the tensor unit's grid of row
parts x column panels and times 20 pipelined steps of each grid through
the executor (host buffers, copies inside every step). Prints JSON.
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

n = m = k = 16384
units = ("gpu0.tc=xpu:dev=0:sms=146:dtype=bf16:elem=2:link=pcie:probe=8192-16384:preroll=20;"
         "gpu0.simt=gpu:dev=0:sms=2:exclusive=1:elem=4:link=pcie:probe=512-2048:preroll=20")
prof = poas.profile_machine(units, "probes=5,repetitions=2,bandwidth_payload=268435456", True, retries=2)
base = json.loads(poas.plan_policy(prof, m, n, k, "overlap"))
hA = torch.empty(m, k).uniform_(-1, 1).pin_memory()
hB = torch.empty(k, n).uniform_(-1, 1).pin_memory()
hA16, hB16 = hA.bfloat16().pin_memory(), hB.bfloat16().pin_memory()
hC = torch.empty(m, n).pin_memory()
io = poas.GemmIO(m=m, n=n, k=k, a_host=hA.data_ptr(), lda_host=k, b_host=hB.data_ptr(), ldb_host=n,
                 c_host=hC.data_ptr(), ldc_host=n, resident=0)
io.a16_host, io.lda16_host = hA16.data_ptr(), k
io.b16_host, io.ldb16_host = hB16.data_ptr(), n
ex = poas.Executor(units + ";overlap=1;pipeline=1")
out = {"base_grid": None, "rows": []}
tc = [d for d in base["devices"] if d["id"] == "gpu0.tc"][0]
out["base_grid"] = [len({t["m"] for t in tc["tiles"]}), len(tc["tiles"])]
import os  # noqa: E402

grids = ((4, 4), (8, 4), (4, 8), (8, 8), (16, 4), (16, 8), (8, 16), (16, 16), (32, 8))
if os.environ.get("E2E_GRID_STAGING_AB"):  # A/B one vs two staging sets, planner's and 16x4 grids
    grids = ((4, 4), (16, 4)) * 3
if os.environ.get("E2E_GRID_LIST"):  # e.g. "16x1,8x2"
    grids = tuple(tuple(int(v) for v in g.split("x")) for g in os.environ["E2E_GRID_LIST"].split(","))
for R, Q in grids:
    s = json.loads(json.dumps(base))
    d = [x for x in s["devices"] if x["id"] == "gpu0.tc"][0]
    pr, pc = d["rows"] // R, n // Q
    d["tiles"] = [{"m": pr, "k": k, "n": pc} for _ in range(R) for _ in range(Q)]
    sched = poas.schedule_roundtrip(json.dumps(s))
    variants = (("two_sets", None), ("one_set", "1")) if os.environ.get("E2E_GRID_STAGING_AB") else (("default", None),)
    row = {"grid": [R, Q]}
    for name, env in variants:
        if env:
            os.environ["POAS_EXEC_PIPE_STAGING"] = env
        else:
            os.environ.pop("POAS_EXEC_PIPE_STAGING", None)
        ex.execute(sched, io, 3)
        t0 = time.perf_counter()
        ex.execute(sched, io, 20)
        ms = (time.perf_counter() - t0) / 20 * 1e3
        row[name] = {"ms_per_step": round(ms, 3), "tflops": round(2 * n ** 3 / ms / 1e9, 1)}
    out["rows"].append(row)
    print(json.dumps(row), file=sys.stderr, flush=True)
print(json.dumps(out))
