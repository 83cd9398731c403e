"""cuBLAS bf16 -> fp32 GEMM target for ncu (timing reference only)."""
import sys

import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
a = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
b = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
c = torch.empty(n, n, device="cuda")
for _ in range(3):
    torch.mm(a, b, out_dtype=torch.float32, out=c)
torch.cuda.synchronize()
