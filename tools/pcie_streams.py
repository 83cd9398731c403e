"""Concurrent H2D + D2H throughput vs copy-stream count (dev tool).

    python tools/pcie_streams.py

1 GiB each way at once (pinned host), split into 64 MiB chunks issued
round-robin on S streams per direction; GB/s per direction. Tells whether
the e2e step's link (one stream per direction) leaves bandwidth unused.
"""
import json

import torch

GiB = 1 << 30
chunk = 64 << 20
h_src = torch.empty(GiB, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(GiB, dtype=torch.uint8).pin_memory()
d_dst = torch.empty(GiB, dtype=torch.uint8, device="cuda")
d_src = torch.empty(GiB, dtype=torch.uint8, device="cuda")
out = {}
for s_in, s_out in ((1, 1), (1, 2), (2, 2), (2, 1), (4, 4)):
    sin = [torch.cuda.Stream() for _ in range(s_in)]
    sout = [torch.cuda.Stream() for _ in range(s_out)]
    best = None
    for _ in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(True)
        e0.record()
        ends = []
        for i in range(GiB // chunk):
            a, b = i * chunk, (i + 1) * chunk
            st = sin[i % s_in]
            st.wait_event(e0)
            with torch.cuda.stream(st):
                d_dst[a:b].copy_(h_src[a:b], non_blocking=True)
            st = sout[i % s_out]
            st.wait_event(e0)
            with torch.cuda.stream(st):
                h_dst[a:b].copy_(d_src[a:b], non_blocking=True)
        ev = []
        for st in sin + sout:
            e = torch.cuda.Event(True)
            e.record(st)
            ev.append(e)
        torch.cuda.synchronize()
        t = max(e0.elapsed_time(e) for e in ev) / 1e3
        best = t if best is None else min(best, t)
    out[f"{s_in}x{s_out}"] = {"ms": round(best * 1e3, 2), "gbs_each_way": round(GiB / best / 1e9, 1)}
print(json.dumps(out))
