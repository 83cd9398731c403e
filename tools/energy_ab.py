"""Sustained A/B of the tensor kernel against cuBLAS (dev tool, timing only).

    python tools/energy_ab.py [N] [seconds] [rounds]

Alternates ~`seconds` of back-to-back launches of each contender, `rounds`
times, and reports per contender: TFLOP/s (CUDA events), joules per GEMM
(NVML total-energy counter), median SM clock and power while it ran. Under
the B200's power cap, J/GEMM decides sustained throughput.
Env POAS_AB_VARIANTS="name:ENV=V,ENV2=V;name2:..." adds variants of our
kernel (env knobs read per launch).
"""
import json
import os
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, os.environ.get("POAS_TREE", str(Path(__file__).resolve().parent.parent)))

import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
secs = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())

a = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
b = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
c = torch.empty(n, n, device="cuda")
poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), n, n, n, 0, 0, n, 1)
poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, n, n, 0, 0, n, 2)
st = torch.cuda.current_stream().cuda_stream


def ours():
    poas.tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, stream=st)


def cublas():
    torch.mm(a, b, out_dtype=torch.float32, out=c)


contenders = {"ours": (ours, {}), "cublas": (cublas, {})}
for spec in filter(None, os.environ.get("POAS_AB_VARIANTS", "").split(";")):
    name, envs = spec.split(":", 1)
    contenders[name] = (ours, dict(kv.split("=", 1) for kv in envs.split(",") if kv))


def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
        time.sleep(0.02)


flop = 2.0 * n ** 3
one = None
res = {k: [] for k in contenders}
for r in range(rounds):
    for name, (fn, env) in contenders.items():
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        fn()
        torch.cuda.synchronize()
        if one is None:
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            one = e0.elapsed_time(e1) / 1e3
        iters = max(3, int(secs / one))
        samples, stop = [], threading.Event()
        th = threading.Thread(target=sample, args=(stop, samples))
        th.start()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        j0 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        j1 = pynvml.nvmlDeviceGetTotalEnergyConsumption(h)
        stop.set(); th.join()
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
        t = e0.elapsed_time(e1) / 1e3 / iters
        clk = sorted(s[0] for s in samples)
        pw = sorted(s[1] for s in samples)
        row = {"round": r, "name": name, "iters": iters, "ms": t * 1e3, "tflops": flop / t / 1e12,
               "j_per_gemm": (j1 - j0) / 1e3 / iters, "sm_mhz_median": clk[len(clk) // 2] if clk else None,
               "power_w_median": pw[len(pw) // 2] if pw else None}
        res[name].append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
        time.sleep(0.5)

summary = {}
for name, rows in res.items():
    summary[name] = {k: sum(r[k] for r in rows) / len(rows) for k in ("tflops", "j_per_gemm", "sm_mhz_median", "power_w_median")}
print(json.dumps({"n": n, "secs": secs, "rounds": rounds, "summary": summary, "rows": res}))
