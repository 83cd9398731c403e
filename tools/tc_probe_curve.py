"""Tensor-unit probe times over a side range (dev tool): what the profiler's
time_gemm sees (pre-rolled, sustained), beside the kernel timed back to
back -- to see where a linear-in-ops model bends.

    python tools/tc_probe_curve.py LO HI STEP [PREROLL_MS]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2209_10245_b200 import poas  # noqa: E402

lo, hi, step = (int(x) for x in sys.argv[1:4])
pre = int(sys.argv[4]) if len(sys.argv) > 4 else 20
u = poas.Unit(f"t=xpu:dev=0:sms=146:dtype=bf16:elem=2:link=hbm:preroll={pre}")
for _ in range(50):
    u.time_gemm(hi)  # warm: the sustained regime
out = []
for side in range(lo, hi + 1, step):
    t = [u.time_gemm(side) for _ in range(3)]
    out.append({"side": side, "ms": [round(x * 1e3, 5) for x in t],
                "tflops": round(2 * side ** 3 / min(t) / 1e12, 1)})
    print(json.dumps(out[-1]), flush=True)
