"""Executor overhead at small sizes (dev tool): per-phase event times of a
resident 1024^3 / 2048^3 run vs the bare kernel."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

units = ("gpu0.tc=xpu:dev=0:sms=146:dtype=bf16:elem=2:link=hbm:probe=8192-16384;"
         "gpu0.simt=gpu:dev=0:sms=2:exclusive=1:elem=4:link=hbm:probe=512-2048")
prof = poas.profile_machine(units, "probes=5,repetitions=2,bandwidth_payload=67108864", True)
ex = poas.Executor(units)
for n in (1024, 2048):
    a16 = torch.randn(n, n, device="cuda").bfloat16()
    b16 = torch.randn(n, n, device="cuda").bfloat16()
    a32 = torch.randn(n, n, device="cuda")
    c = torch.empty(n, n, device="cuda")
    io = poas.GemmIO(m=n, n=n, k=n, a_dev=a32.data_ptr(), lda_dev=n, b_dev=a32.data_ptr(), ldb_dev=n,
                     a16_dev=a16.data_ptr(), lda16_dev=n, b16_dev=b16.data_ptr(), ldb16_dev=n,
                     c_dev=c.data_ptr(), ldc_dev=n, resident=1)
    sched = poas.plan_standalone(prof, "gpu0.tc", n, n, n)
    ex.execute(sched, io, 3)
    rep = ex.execute(sched, io, 20)
    s = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        poas.tc_gemm(2, n, n, n, a16.data_ptr(), n, b16.data_ptr(), n, c.data_ptr(), n, num_ctas=146, stream=s)
    e1.record()
    torch.cuda.synchronize()
    d = [x for x in rep["devices"] if x["id"] == "gpu0.tc"][0]
    print(json.dumps({"n": n, "measured_makespan_us": rep["measured_makespan"] * 1e6,
                      "compute_us": d["compute"]["measured"] * 1e6,
                      "copy_in_us": d["copy_in"]["measured"] * 1e6,
                      "finish_us": d["finish"]["measured"] * 1e6,
                      "bare_kernel_us": e0.elapsed_time(e1) / 20 * 1e3,
                      "wall_us": rep["measured_wall"] * 1e6}))
