"""Dynamic warm-up vs the timed chained run at C5 sizes (dev tool)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

units = ("gpu0.tc=xpu:dev=0:sms=146:dtype=bf16:elem=2:link=hbm:probe=8192-16384;"
         "gpu0.simt=gpu:dev=0:sms=2:exclusive=1:elem=4:link=hbm:probe=512-2048")
prof = poas.profile_machine(units, "probes=9,repetitions=3,bandwidth_payload=268435456", True)
ex = poas.Executor(units)
for n in (4096, 8192):
    a16 = torch.randn(n, n, device="cuda").bfloat16()
    b16 = torch.randn(n, n, device="cuda").bfloat16()
    a32 = torch.randn(n, n, device="cuda")
    c = torch.empty(n, n, device="cuda")
    io = poas.GemmIO(m=n, n=n, k=n, a_dev=a32.data_ptr(), lda_dev=n, b_dev=a32.data_ptr(), ldb_dev=n,
                     a16_dev=a16.data_ptr(), lda16_dev=n, b16_dev=b16.data_ptr(), ldb16_dev=n,
                     c_dev=c.data_ptr(), ldc_dev=n, resident=1)
    dyn = ex.run_dynamic(prof, n, n, n, io, iterations=15, alpha=1.0, replan_threshold_pct=2.0)
    for it in dyn["iterations"]:
        print(n, it["iteration"], it["replanned"], it["rows"], round(it["predicted_makespan"] * 1e6, 1),
              round(it["measured_makespan"] * 1e6, 1), round(it["makespan_error_pct"], 2))
    sched = poas.schedule_roundtrip(json.dumps(dyn["schedule"]))
    rep = ex.execute(sched, io, 15)
    d = {x["id"]: (round(x["compute"]["measured"] * 1e6, 1), round(x["compute"]["predicted"] * 1e6, 1),
                   round(x["copy_in"]["predicted"] * 1e6, 1), round(x["copy_out"]["predicted"] * 1e6, 1))
         for x in rep["devices"]}
    print(n, "timed", round(rep["predicted_makespan"] * 1e6, 1), round(rep["measured_makespan"] * 1e6, 1),
          round(rep["makespan_error_pct"], 2), d, [round(x * 1e6, 1) for x in rep["repeat_makespans"]])
