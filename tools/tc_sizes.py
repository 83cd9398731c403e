"""Back-to-back tensor-kernel launch times over square sizes (dev tool).

    python tools/tc_sizes.py [sizes...]

Prints one JSON line: per size, the mean time of 64 back-to-back launches
(after 16 warm-up launches) for the default variant and each forced one.
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, os.environ.get("POAS_TREE", str(Path(__file__).resolve().parent.parent)))

import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

sizes = [int(x) for x in sys.argv[1:]] or [1024, 2048, 3072, 4096, 8192]
variants = os.environ.get("POAS_SIZES_VARIANTS", "default,2cta,2cta512").split(",")
st = torch.cuda.current_stream().cuda_stream
out = {"tree": os.environ.get("POAS_TREE", "."), "rows": []}
for n in sizes:
    a = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    b = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(n, n, device="cuda")
    poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), n, n, n, 0, 0, n, 1)
    poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, n, n, 0, 0, n, 2)
    row = {"n": n}
    for v in variants:
        if v == "default":
            os.environ.pop("POAS_TC_KERNEL", None)
        else:
            os.environ["POAS_TC_KERNEL"] = v
        fn = lambda: poas.tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, stream=st)  # noqa: E731
        reps = 64 if n <= 4096 else 16
        for _ in range(16):
            fn()
        torch.cuda.synchronize()
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / reps * 1e3
            best = t if best is None else min(best, t)
        row[v] = {"us": round(best, 2), "tflops": round(2 * n ** 3 / best / 1e6, 1)}
    os.environ.pop("POAS_TC_KERNEL", None)
    ref = lambda: torch.mm(a, b, out_dtype=torch.float32, out=c)  # noqa: E731
    for _ in range(16):
        ref()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        ref()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps * 1e3
    row["cublas"] = {"us": round(t, 2), "tflops": round(2 * n ** 3 / t / 1e6, 1)}
    out["rows"].append(row)
    print(json.dumps(row), file=sys.stderr, flush=True)
print(json.dumps(out))
