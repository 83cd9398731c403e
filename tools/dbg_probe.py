"""Probe vs timed-step diagnosis at small sizes (dev tool; profiles/r02_fused).

    python tools/dbg_probe.py

For 2048^3 and 4096^3: the tensor unit's fitted model at its lent budget
(two-point and nine-point probe sets) against executor runs of 1 / 42 / 256
graph-replayed repeats and Python-loop launches.
"""
import sys, json, time
sys.path.insert(0, '.')
import torch
from paper_2209_10245_b200 import poas
sys.path.insert(0, 'tools')
import sweep as sw
for n in (2048, 4096):
    lo, hi = sw.tc_probe_range(n)
    lent = f"gpu0.tc=xpu:dev=0:sms=148:dtype=bf16:elem=2:link=hbm:probe={lo}-{hi}:preroll=20"
    for prof_s in (sw.PROF_TC, sw.PROF):
        p = poas.profile_machine(lent, prof_s, True, retries=2)
        f = {l.split()[0]: l.split()[1] for l in p.splitlines() if len(l.split()) == 2}
        slope, icpt = float(f['slope']), float(f['intercept'])
        pred = slope * n**3 + icpt
        print(n, prof_s[:8], 'slope', slope, 'icpt', icpt, 'pred_us', pred * 1e6)
    d = sw.operands(n); io = sw.io_for(n, d)
    units = (f"gpu0.tc=xpu:dev=0:sms=146:dtype=bf16:elem=2:link=hbm:probe={lo}-{hi}:preroll=20;"
             "gpu0.simt=gpu:dev=0:sms=2:exclusive=1:elem=4:link=hbm:probe=512-2048")
    ex = poas.Executor(units)
    prof = poas.profile_machine(units, sw.PROF, True, retries=2)
    sched = poas.plan_policy(prof, n, n, n, "best-subset")
    for reps in (1, 42, 256):
        ex.execute(sched, io, reps)
        r = ex.execute(sched, io, reps)
        print(n, 'exec reps', reps, 'meas_us', r['measured_makespan'] * 1e6)
    st = torch.cuda.current_stream().cuda_stream
    fn = lambda: poas.tc_gemm(2, n, n, n, d["A16"].data_ptr(), n, d["B16"].data_ptr(), n, d["C"].data_ptr(), n, stream=st)
    for reps in (1, 6, 64):
        for _ in range(20): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        print(n, 'python reps', reps, 'us', e0.elapsed_time(e1) / reps * 1e3)
