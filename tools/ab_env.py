"""A/B of two tc_gemm env settings under sustained load, ABBA order (dev
tool): each block = 10 back-to-back 16384^3 launches; medians per variant.

    python tools/ab_env.py "K:V,K:V" "K:V" [rounds]
"""
import json
import os
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402

KEYS = ("POAS_TC_HINT_A", "POAS_TC_HINT_B", "POAS_TC_HINT_C", "POAS_TC_GROUP", "POAS_TC_SCHED", "POAS_TC_KERNEL",
        "POAS_TC_KSERP")


def env_of(spec):
    return dict(kv.split(":", 1) for kv in spec.split(",") if kv)


def main():
    a_spec, b_spec = sys.argv[1], sys.argv[2]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 6
    n = int(os.environ.get("AB_N", "16384"))
    A = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    B = torch.empty(n, n, device="cuda", dtype=torch.bfloat16)
    C = torch.empty(n, n, device="cuda")
    poas.fill_uniform(poas.DTYPE_BF16, A.data_ptr(), n, n, n, 0, 0, n, 1)
    poas.fill_uniform(poas.DTYPE_BF16, B.data_ptr(), n, n, n, 0, 0, n, 2)
    s = torch.cuda.current_stream().cuda_stream
    res = {"A": [], "B": []}

    def block(spec):
        for k in KEYS:
            os.environ.pop(k, None)
        os.environ.update(env_of(spec))
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10):
            poas.tc_gemm(2, n, n, n, A.data_ptr(), n, B.data_ptr(), n, C.data_ptr(), n, stream=s)
        e1.record()
        e1.synchronize()
        return 2 * n ** 3 / (e0.elapsed_time(e1) / 10) / 1e9

    block(a_spec)
    block(b_spec)
    for r in range(rounds):
        order = ("A", "B", "B", "A") if r % 2 == 0 else ("B", "A", "A", "B")
        for v in order:
            res[v].append(round(block(a_spec if v == "A" else b_spec), 1))
    print(json.dumps({"A": a_spec, "B": b_spec, "A_median": statistics.median(res["A"]),
                      "B_median": statistics.median(res["B"]), "runs": res}))


if __name__ == "__main__":
    main()
