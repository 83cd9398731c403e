"""ncu target: one tc_gemm (row-major B) or tc_gemm_panels (P panels) launch (dev tool).

    python tools/ncu_panels.py M N K P      # P = 1: row-major B
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

m, n, k, P = (int(x) for x in sys.argv[1:5])
a = torch.empty(m, k, device="cuda", dtype=torch.bfloat16)
b = torch.empty(k, n, device="cuda", dtype=torch.bfloat16)
poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), k, m, k, 0, 0, k, 1)
poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, k, n, 0, 0, n, 2)
c = torch.empty(m, n, device="cuda")
np_ = n // P
bp = torch.stack([b[:, p * np_:(p + 1) * np_] for p in range(P)]).contiguous() if P > 1 else b
for _ in range(3):
    if P > 1:
        poas.tc_gemm_panels(2, m, n, k, a.data_ptr(), k, bp.data_ptr(), np_, c.data_ptr(), n, P)
    else:
        poas.tc_gemm(2, m, n, k, a.data_ptr(), k, b.data_ptr(), n, c.data_ptr(), n)
torch.cuda.synchronize()
