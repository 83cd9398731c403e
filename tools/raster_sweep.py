"""Raster-group / kernel-variant sweep of the tensor unit (dev tool).

    python tools/raster_sweep.py  ->  JSON {variant: {N: {group: TFLOP/s}}}
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402


def run(n, iters=6):
    a = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    b = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(n, n, device="cuda")
    poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), n, n, n, 0, 0, n, 1)
    poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, n, n, 0, 0, n, 2)
    s = torch.cuda.current_stream().cuda_stream
    res = {}
    for variant in ("2cta", "1cta"):
        os.environ["POAS_TC_KERNEL"] = variant
        res[variant] = {}
        for group in (1, 2, 4, 8, 16, 32, 64):
            os.environ["POAS_TC_GROUP"] = str(group)
            f = lambda: poas.tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n,  # noqa
                                     stream=s)
            f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(iters):
                f()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / iters
            res[variant][group] = round(2 * n ** 3 / ms / 1e9, 1)
    os.environ.pop("POAS_TC_GROUP", None)
    os.environ.pop("POAS_TC_KERNEL", None)
    return res


if __name__ == "__main__":
    sizes = [int(x) for x in sys.argv[1:]] or [8192, 16384, 32768]
    out = {}
    for n in sizes:
        out[n] = run(n)
        print(n, json.dumps(out[n]), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))
