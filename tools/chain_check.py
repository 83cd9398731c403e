"""Single-repeat executes vs one chained execute (dev tool): per-repeat
measured makespans of the same schedule."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

units = ("gpu0.tc=xpu:dev=0:sms=146:dtype=bf16:elem=2:link=hbm:probe=8192-16384;"
         "gpu0.simt=gpu:dev=0:sms=2:exclusive=1:elem=4:link=hbm:probe=512-2048")
prof = poas.profile_machine(units, "probes=5,repetitions=2,bandwidth_payload=67108864", True)
ex = poas.Executor(units)
for n in (2048, 4096, 8192):
    a16 = torch.randn(n, n, device="cuda").bfloat16()
    b16 = torch.randn(n, n, device="cuda").bfloat16()
    a32 = torch.randn(n, n, device="cuda")
    c = torch.empty(n, n, device="cuda")
    io = poas.GemmIO(m=n, n=n, k=n, a_dev=a32.data_ptr(), lda_dev=n, b_dev=a32.data_ptr(), ldb_dev=n,
                     a16_dev=a16.data_ptr(), lda16_dev=n, b16_dev=b16.data_ptr(), ldb16_dev=n,
                     c_dev=c.data_ptr(), ldc_dev=n, resident=1)
    sched = poas.plan_standalone(prof, "gpu0.tc", n, n, n)
    ex.execute(sched, io, 3)
    single = [ex.execute(sched, io, 1)["measured_makespan"] * 1e6 for _ in range(10)]
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    chained_rep = ex.execute(sched, io, 10)
    e1.record()
    torch.cuda.synchronize()
    chained = chained_rep["repeat_makespans"]
    total_chained_us = e0.elapsed_time(e1) * 1e3 / 10
    e0.record()
    for _ in range(10):
        ex.execute(sched, io, 1)
    e1.record()
    torch.cuda.synchronize()
    total_single_us = e0.elapsed_time(e1) * 1e3 / 10
    devs = {d["id"]: (d["compute"]["measured"] * 1e6, d["finish"]["measured"] * 1e6,
                      d["finish"]["predicted"] * 1e6) for d in chained_rep["devices"]}
    print(json.dumps({"n": n, "single_us": [round(x, 1) for x in single],
                      "chained_us": [round(x * 1e6, 1) for x in chained],
                      "single_median": statistics.median(single),
                      "chained_median": statistics.median(chained) * 1e6,
                      "events_per_repeat_chained_us": total_chained_us,
                      "events_per_repeat_single_us": total_single_us,
                      "chained_devices_compute_finish_pred_us": devs,
                      "predicted_us": chained_rep["predicted_makespan"] * 1e6}))
