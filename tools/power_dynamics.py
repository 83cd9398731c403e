"""Per-repeat makespans of consecutive K-step blocks of the 16384^3 resident
step (dev tool): how the power-capped clock moves the step time over
seconds. Prints JSON: [[block0 repeat makespans ms], ...] + NVML clocks."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

try:
    import pynvml
    pynvml.nvmlInit()
    H = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:
    H = None

n = 16384
units = "gpu0.tc=xpu:dev=0:sms=146:dtype=bf16:elem=2:link=hbm:probe=8192-16384;gpu0.simt=gpu:dev=0:sms=2:exclusive=1:elem=4:link=hbm:probe=512-2048"
prof = poas.profile_machine(units, "probes=5,repetitions=2,bandwidth_payload=67108864", True)
sched = poas.plan_standalone(prof, "gpu0.tc", n, n, n)
A = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
B = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
C = torch.empty(n, n, device="cuda")
poas.fill_uniform(poas.DTYPE_BF16, A.data_ptr(), n, n, n, 0, 0, n, 1)
poas.fill_uniform(poas.DTYPE_BF16, B.data_ptr(), n, n, n, 0, 0, n, 2)
io = poas.GemmIO(m=n, n=n, k=n, a16_dev=A.data_ptr(), lda16_dev=n, b16_dev=B.data_ptr(), ldb16_dev=n,
                 c_dev=C.data_ptr(), ldc_dev=n, resident=1)
ex = poas.Executor(units)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 10
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 20
gap = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
out = []
t_start = time.perf_counter()
for b in range(blocks):
    rep = ex.execute(sched, io, K)
    clk = pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM) if H else None
    out.append({"t": round(time.perf_counter() - t_start, 3), "mean_ms": round(rep["measured_makespan"] * 1e3, 3),
                "repeats_ms": [round(x * 1e3, 2) for x in rep["repeat_makespans"]], "sm_mhz_after": clk})
    time.sleep(gap)
print(json.dumps(out, indent=0))
