"""Overlapped e2e at 16384^3 (bf16 host A/B, fp32 C) for hand-set grids of
row parts x column panels (dev tool): the streamed launch's measured step
per grid. Prints JSON."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

n = m = k = 16384
units = "gpu0.tc=xpu:dev=0:sms=148:dtype=bf16:elem=2:link=pcie:probe=8192-16384"
sa, sb = poas.stream_seed(20261017, "A"), poas.stream_seed(20261017, "B")
hA = torch.empty(m, k, dtype=torch.float32, pin_memory=True)
hB = torch.empty(k, n, dtype=torch.float32, pin_memory=True)
poas.fill_uniform_host(hA.data_ptr(), k, m, k, 0, 0, k, sa)
poas.fill_uniform_host(hB.data_ptr(), n, k, n, 0, 0, n, sb)
hA16 = hA.bfloat16().pin_memory()
hB16 = hB.bfloat16().pin_memory()
del hA, hB
hC = torch.empty(m, n, dtype=torch.float32, pin_memory=True)
prof = poas.profile_machine(units, "probes=5,repetitions=2,bandwidth_payload=268435456", True)
base = json.loads(poas.plan_policy(prof, m, n, k, "overlap"))
io = poas.GemmIO(m=m, n=n, k=k, c_host=hC.data_ptr(), ldc_host=n, resident=0,
                 a16_host=hA16.data_ptr(), lda16_host=k, b16_host=hB16.data_ptr(), ldb16_host=n)
ex = poas.Executor(units + ";overlap=1")
out = {}
grids = [(int(g.split("x")[0]), int(g.split("x")[1])) for g in sys.argv[1].split(",")] if len(sys.argv) > 1 else [(64, 1), (32, 2), (32, 4), (16, 8), (32, 8), (64, 8), (16, 16), (32, 16)]
for R, Q in grids:
    s = dict(base)
    dev = dict(s["devices"][0])
    rp, cp = [m // R] * R, [n // Q] * Q
    dev["tiles"] = [{"m": r, "k": k, "n": w} for r in rp for w in cp]
    s["devices"] = [dev] + s["devices"][1:]
    txt = poas.schedule_roundtrip(json.dumps(s))
    ex.execute(txt, io, 1)
    rep = ex.execute(txt, io, 4)
    d = rep["devices"][0]
    out[f"{R}x{Q}"] = {"ms": round(rep["measured_makespan"] * 1e3, 3),
                       "tflops": round(2 * m * n * k / rep["measured_makespan"] / 1e12, 1),
                       "copy_in_ms": round(d["copy_in"]["measured"] * 1e3, 2),
                       "copy_out_ms": round(d["copy_out"]["measured"] * 1e3, 2)}
    print(f"{R}x{Q}", out[f"{R}x{Q}"], file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
