"""Small-size tensor GEMM study (dev tool): our tc_gemm vs cuBLAS (bf16 in,
fp32 out) at N in {512..4096}, CUDA events, (a) back-to-back launches
(steady state) and (b) one launch after a sync (latency). Prints JSON.

    python tools/small_gemm.py [iters]
    python tools/small_gemm.py one N ours|cublas   # ncu target: 3 warm-up + 1
"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402


def operands(n):
    a = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    b = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), n, n, n, 0, 0, n, 1)
    poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, n, n, 0, 0, n, 2)
    return a, b, torch.empty(n, n, device="cuda")


def fns(n):
    a, b, c = operands(n)
    s = torch.cuda.current_stream().cuda_stream

    def ours():
        poas.tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, stream=s)

    def cublas():
        torch.mm(a, b, out_dtype=torch.float32, out=c)

    return {"ours": ours, "cublas": cublas}


def timed(fn, iters, back_to_back):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    if back_to_back:
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters * 1e3
    out = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(out)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        n = int(sys.argv[2])
        f = fns(n)[sys.argv[3]]
        for _ in range(4):
            f()
        torch.cuda.synchronize()
        sys.exit(0)
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    res = {}
    for n in (512, 1024, 2048, 3072, 4096):
        f = fns(n)
        row = {}
        for name, fn in f.items():
            b2b = timed(fn, iters, True)
            one = timed(fn, iters, False)
            row[name] = {"b2b_us": round(b2b, 2), "single_us": round(one, 2),
                         "b2b_tflops": round(2 * n**3 / (b2b * 1e-6) / 1e12, 1),
                         "single_tflops": round(2 * n**3 / (one * 1e-6) / 1e12, 1)}
        res[n] = row
    print(json.dumps(res, indent=1))
