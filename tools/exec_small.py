"""Executor step vs the bare tensor kernel at small sizes (dev tool).

    python tools/exec_small.py [sizes...]

Per size: a one-unit resident plan of the tensor unit (146 SMs + 2 lent)
run through the executor for 256 repeats (CUDA-graph replay; also with
POAS_EXEC_GRAPH=0), beside 256 back-to-back tc_gemm launches from Python
on every SM. Mean microseconds per GEMM; alternating, best of 3.
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

UNITS = ("gpu0.tc=xpu:dev=0:sms=146:dtype=bf16:elem=2:link=hbm:probe=2048-4096;"
         "gpu0.simt=gpu:dev=0:sms=2:exclusive=1:elem=4:link=hbm:probe=256-512")
prof = poas.profile_machine(UNITS, "probes=4,repetitions=2,bandwidth_payload=16777216", True)
ex = poas.Executor(UNITS)
out = []
for n in [int(x) for x in sys.argv[1:]] or [1024, 2048, 4096]:
    a = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    b = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(n, n, device="cuda")
    poas.fill_uniform(poas.DTYPE_BF16, a.data_ptr(), n, n, n, 0, 0, n, 1)
    poas.fill_uniform(poas.DTYPE_BF16, b.data_ptr(), n, n, n, 0, 0, n, 2)
    sched = poas.plan_standalone(prof, "gpu0.tc", n, n, n)
    io = poas.GemmIO(m=n, n=n, k=n, a16_dev=a.data_ptr(), lda16_dev=n, b16_dev=b.data_ptr(), ldb16_dev=n,
                     c_dev=c.data_ptr(), ldc_dev=n, resident=1)
    st = torch.cuda.current_stream().cuda_stream
    res = {"n": n, "kernel": poas.tc_kernel_name(n, n, n)}
    best = {}
    for _ in range(3):
        for mode in ("graph", "nograph", "python"):
            if mode == "python":
                for _ in range(16):
                    poas.tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, stream=st)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record()
                for _ in range(256):
                    poas.tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, stream=st)
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 256 * 1e3
            else:
                if mode == "nograph":
                    os.environ["POAS_EXEC_GRAPH"] = "0"
                else:
                    os.environ.pop("POAS_EXEC_GRAPH", None)
                ex.execute(sched, io, 256)
                rep = ex.execute(sched, io, 256)
                t = rep["measured_makespan"] * 1e6
            best[mode] = min(best.get(mode, 1e30), t)
    os.environ.pop("POAS_EXEC_GRAPH", None)
    res.update({k: round(v, 2) for k, v in best.items()})
    res["tflops"] = {k: round(2 * n ** 3 / v / 1e6, 1) for k, v in best.items()}
    out.append(res)
    print(json.dumps(res), file=sys.stderr, flush=True)
print(json.dumps(out))
