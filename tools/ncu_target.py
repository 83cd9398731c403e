"""Single-kernel targets for ncu captures and micro-timing (dev tool).

    python tools/ncu_target.py tc   [N]        # 2 warm-up + 1 tc_gemm launch at N^3
    python tools/ncu_target.py simt ROWS [N] [SMS]  # skinny CUDA-core share
    python tools/ncu_target.py micro            # CUDA-event timings, prints JSON
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, os.environ.get("POAS_TREE", str(Path(__file__).resolve().parent.parent)))

import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402


def tc(n, sms=0, iters=1, warm=2):
    a = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    b = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(n, n, device="cuda")
    poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), n, n, n, 0, 0, n, 1)
    poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, n, n, 0, 0, n, 2)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(warm):
        poas.tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, num_ctas=sms, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        poas.tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, num_ctas=sms, stream=s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def simt(rows, n, sms, iters=1, warm=1, exclusive=True):
    a = torch.empty(rows, n, device="cuda")
    b = torch.empty(n, n, device="cuda")
    c = torch.empty(rows, n, device="cuda")
    poas.fill_uniform(poas.DTYPE_F32, a.data_ptr(), n, rows, n, 0, 0, n, 1)
    poas.fill_uniform(poas.DTYPE_F32, b.data_ptr(), n, n, n, 0, 0, n, 2)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(warm):
        poas.simt_gemm(rows, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, num_ctas=sms,
                       exclusive=exclusive, stream=s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        poas.simt_gemm(rows, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, num_ctas=sms,
                       exclusive=exclusive, stream=s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "tc":
        n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
        print(tc(n))
    elif what == "simt":
        rows = int(sys.argv[2])
        n = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
        sms = int(sys.argv[4]) if len(sys.argv) > 4 else 2
        print(simt(rows, n, sms, exclusive=sms > 0))
    else:
        out = {"tc": {}, "simt_2sm": {}, "simt_all": {}}
        for n in (4096, 8192, 16384):
            ms = tc(n, iters=5)
            out["tc"][n] = {"ms": ms, "tflops": 2 * n**3 / ms / 1e9}
        for sms in (146, 144, 140):
            ms = tc(16384, sms=sms, iters=5)
            out["tc"][f"16384@{sms}sm"] = {"ms": ms, "tflops": 2 * 16384**3 / ms / 1e9}
        for rows in (4, 8, 16, 24, 64, 128, 512):
            ms = simt(rows, 16384, 2, iters=2)
            out["simt_2sm"][rows] = {"ms": ms, "tflops": 2 * rows * 16384**2 / ms / 1e9,
                                     "b_gbs": 16384**2 * 4 / ms / 1e6}
        for n in (2048, 4096, 8192):
            ms = simt(n, n, 0, iters=2, exclusive=False)
            out["simt_all"][n] = {"ms": ms, "tflops": 2 * n**3 / ms / 1e9}
        print(json.dumps(out, indent=1))
