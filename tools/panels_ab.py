"""Panel-major B (the multi-GPU consumer) vs row-major B, one GPU (dev tool).

    python tools/panels_ab.py [m] [n] [k]

Back-to-back launches of tc_gemm (row-major B) and tc_gemm_panels with P
panels (flags set), default variant; TFLOP/s per P, alternating, best of 3.
The C4 shape per GPU at 8 GPUs is 8192 x 8192 x 8192 with P = 16.
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
k = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
a = torch.empty(m, k, device="cuda", dtype=torch.bfloat16)
b = torch.empty(k, n, device="cuda", dtype=torch.bfloat16)
poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), k, m, k, 0, 0, k, 1)
poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, k, n, 0, 0, n, 2)
c = torch.empty(m, n, device="cuda")
st = torch.cuda.current_stream().cuda_stream
fns = {"rowmajor": lambda: poas.tc_gemm(2, m, n, k, a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n, stream=st)}
bps = {}
for P in (4, 8, 16):
    np_ = n // P
    bps[P] = torch.stack([b[:, p * np_:(p + 1) * np_] for p in range(P)]).contiguous()
    flags = torch.ones(P, dtype=torch.int32, device="cuda")
    bps[(P, "f")] = flags
    fns[f"panels{P}"] = (lambda P=P, np_=np_: poas.tc_gemm_panels(
        2, m, n, k, a.data_ptr(), k, bps[P].data_ptr(), np_, c.data_ptr(), n, P,
        flags=bps[(P, "f")].data_ptr(), epoch=1, stream=st))
    fns[f"panels{P}_noflags"] = (lambda P=P, np_=np_: poas.tc_gemm_panels(
        2, m, n, k, a.data_ptr(), k, bps[P].data_ptr(), np_, c.data_ptr(), n, P, stream=st))
iters = 30
best = {}
for _ in range(3):
    for name, fn in fns.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / iters
        best[name] = min(best.get(name, 1e9), t)
print(json.dumps({"shape": [m, n, k], "tflops": {k_: round(2 * m * n * k / v / 1e9, 1) for k_, v in best.items()}}))
