"""Tensor-unit variant comparison under sustained load (dev tool).

Variants (env settings of tc_gemm) are interleaved in rounds so power and
thermal drift hit all of them alike; each timing records the SM clock and
throttle reasons (pynvml). cuBLAS (torch.mm bf16 -> fp32) runs beside them
as the library reference.

    python tools/raster_sweep.py [--rounds R] [--variants NAME=K:V,K:V;...] [N ...]  ->  JSON
"""
import argparse
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

ENV_KEYS = ("POAS_TC_KERNEL", "POAS_TC_GROUP", "POAS_TC_SCHED", "POAS_TC_RASTER")
DEFAULT_VARIANTS = {
    "default": {},  # tc_gemm's own choice of kernel / scheduler for the size
    "2cta:dynamic": {"POAS_TC_KERNEL": "2cta", "POAS_TC_SCHED": "dynamic"},
    "2cta:wave": {"POAS_TC_KERNEL": "2cta", "POAS_TC_SCHED": "wave"},
    "1cta:dynamic": {"POAS_TC_KERNEL": "1cta", "POAS_TC_SCHED": "dynamic"},
    "1cta:wave": {"POAS_TC_KERNEL": "1cta", "POAS_TC_SCHED": "wave"},
    "cublas": None,
}


def clocks():
    if NV is None:
        return None, None
    return (pynvml.nvmlDeviceGetClockInfo(NV, pynvml.NVML_CLOCK_SM),
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(NV))


def parse_variants(text):
    out = {}
    for item in text.split(";"):
        name, _, spec = item.partition("=")
        if spec == "cublas":
            out[name] = None
            continue
        out[name] = dict(kv.split(":", 1) for kv in spec.split(",") if kv)
    return out


def bench(n, variants, rounds=3, iters=8):
    a = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    b = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(n, n, device="cuda")
    c_lib = torch.empty(n, n, device="cuda")
    poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), n, n, n, 0, 0, n, 1)
    poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, n, n, 0, 0, n, 2)
    s = torch.cuda.current_stream().cuda_stream
    res = {name: [] for name in variants}
    for _ in range(rounds):
        for name, env in variants.items():
            for key in ENV_KEYS:
                os.environ.pop(key, None)
            if env is None:
                f = lambda: torch.mm(a, b, out_dtype=torch.float32, out=c_lib)  # noqa: E731
            else:
                os.environ.update(env)
                f = lambda: poas.tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n,  # noqa: E731
                                         c.data_ptr(), n, stream=s)
            for _ in range(2):
                f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(iters):
                f()
            e1.record()
            e1.synchronize()
            clk, why = clocks()
            ms = e0.elapsed_time(e1) / iters
            res[name].append((round(2 * n ** 3 / ms / 1e9, 1), clk, why))
    for key in ENV_KEYS:
        os.environ.pop(key, None)
    return {k: {"tflops_median": statistics.median(x[0] for x in v), "runs": v} for k, v in res.items()}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("sizes", nargs="*", type=int)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--variants", default=None)
    args = ap.parse_args()
    variants = parse_variants(args.variants) if args.variants else DEFAULT_VARIANTS
    out = {}
    for n in args.sizes or [8192, 16384, 32768]:
        out[n] = bench(n, variants, args.rounds)
        print(n, json.dumps({k: v["tflops_median"] for k, v in out[n].items()}), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))
