"""Tensor-unit variant / raster-group comparison with clock sampling (dev tool).

Variants are interleaved in rounds so power/thermal drift hits all of them
alike; each timing records the SM clock and throttle reasons (pynvml).

    python tools/raster_sweep.py [N ...]  ->  JSON
"""
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

try:
    import pynvml

    pynvml.nvmlInit()
    NV = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:  # pragma: no cover
    NV = None


def clocks():
    if NV is None:
        return None, None
    return (pynvml.nvmlDeviceGetClockInfo(NV, pynvml.NVML_CLOCK_SM),
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(NV))


# (kernel, raster group, tile scheduler)
VARIANTS = [("2cta", 8, "dynamic"), ("2cta", 8, "static"), ("2cta", 16, "dynamic"),
            ("1cta", 16, "dynamic"), ("1cta", 16, "static"), ("cublas", 0, "")]


def bench(n, rounds=3, iters=8):
    a = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    b = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(n, n, device="cuda")
    poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), n, n, n, 0, 0, n, 1)
    poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, n, n, 0, 0, n, 2)
    s = torch.cuda.current_stream().cuda_stream
    c16 = torch.empty(n, n, device="cuda")
    res = {f"{v}:{g}:{y}": [] for v, g, y in VARIANTS}
    for _ in range(rounds):
        for v, g, y in VARIANTS:
            if v == "cublas":
                f = lambda: torch.mm(a, b, out_dtype=torch.float32, out=c16)  # noqa: E731
            else:
                os.environ["POAS_TC_KERNEL"] = v
                os.environ["POAS_TC_GROUP"] = str(g)
                os.environ["POAS_TC_SCHED"] = y
                f = lambda: poas.tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n,  # noqa: E731
                                         c.data_ptr(), n, stream=s)
            for _ in range(2):
                f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for i in range(iters):
                f()
            e1.record()
            e1.synchronize()
            clk, why = clocks()
            ms = e0.elapsed_time(e1) / iters
            res[f"{v}:{g}:{y}"].append((round(2 * n ** 3 / ms / 1e9, 1), clk, why))
    os.environ.pop("POAS_TC_GROUP", None)
    os.environ.pop("POAS_TC_KERNEL", None)
    os.environ.pop("POAS_TC_SCHED", None)
    return {k: {"tflops_median": statistics.median(x[0] for x in v), "runs": v} for k, v in res.items()}


if __name__ == "__main__":
    sizes = [int(x) for x in sys.argv[1:]] or [8192, 16384, 32768]
    out = {}
    for n in sizes:
        out[n] = bench(n)
        print(n, json.dumps({k: v["tflops_median"] for k, v in out[n].items()}), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))
