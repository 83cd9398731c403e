"""Per-GPU compute side of the N > 1 bench step, measured on one GPU (dev
tool): the tensor GEMM at 16384^3 on 146 SMs with row-major B (the N = 1
step) vs panel-major B in one tc_gemm_panels launch (flags already set) on
146 and on 140 SMs (TC_SMS_MULTI: 8 SMs left to NCCL), vs per-panel
launches (the event path). CUDA events, alternating. Prints JSON."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

n = 16384
P = 8
np_ = n // P
a = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
b = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), n, n, n, 0, 0, n, 1)
poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, n, n, 0, 0, n, 2)
bp = torch.stack([b[:, p * np_:(p + 1) * np_] for p in range(P)]).contiguous()
c = torch.empty(n, n, device="cuda")
flags = torch.ones(P, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def rowmajor(sms):
    return lambda: poas.tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n,
                                num_ctas=sms, stream=s)


def panels(sms):
    return lambda: poas.tc_gemm_panels(2, n, n, n, a.data_ptr(), n, bp.data_ptr(), np_, c.data_ptr(), n, P,
                                       flags=flags.data_ptr(), epoch=1, num_ctas=sms, stream=s)


def per_panel(sms):
    def f():
        for p in range(P):
            poas.tc_gemm(2, n, np_, n, a.data_ptr(), n, bp[p].data_ptr(), np_, c[:, p * np_:].data_ptr(), n,
                         num_ctas=sms, stream=s)
    return f


cases = {"rowmajor_146": rowmajor(146), "panels_one_launch_146": panels(146),
         "panels_one_launch_140": panels(140), "per_panel_launches_140": per_panel(140)}
for f in cases.values():
    f()
torch.cuda.synchronize()
times = {k: [] for k in cases}
for _ in range(5):
    for k, f in cases.items():
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(3):
            f()
        e1.record()
        torch.cuda.synchronize()
        times[k].append(e0.elapsed_time(e1) / 3)
out = {k: {"ms": round(statistics.median(v), 3), "tflops": round(2 * n ** 3 / statistics.median(v) / 1e9, 1)}
       for k, v in times.items()}
print(json.dumps(out, indent=1))
