"""The CUDA-core kernel beside cuBLAS SGEMM (fp32, TF32 off), every SM,
alternating launches (same power state); each variant of POAS_SIMT_TILE in
its own process (the variant is read per launch, so one process is enough).

    python tools/simt_check.py [N ...]     -> JSON lines
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2209_10245_b200 import poas  # noqa: E402


def ev(fn, it):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e-3


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [4096, 8192]
    torch.backends.cuda.matmul.allow_tf32 = False
    for n in sizes:
        a = torch.empty(n, n, device="cuda")
        b = torch.empty(n, n, device="cuda")
        c = torch.empty(n, n, device="cuda")
        poas.fill_uniform(0, a.data_ptr(), n, n, n, 0, 0, n, 1)
        poas.fill_uniform(0, b.data_ptr(), n, n, n, 0, 0, n, 2)
        st = torch.cuda.current_stream().cuda_stream
        res = {"n": n}
        for variant in ("ffma2", "ffma2k32", "ffma2k16j", "ffma2k16"):
            os.environ["POAS_SIMT_TILE"] = variant
            ours = lambda: poas.simt_gemm(n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n,  # noqa
                                          stream=st)
            ours()
            torch.cuda.synchronize()
            ref = (a.double() @ b.double())
            err = float((c.double() - ref).norm() / ref.norm())
            c_lib = torch.empty(n, n, device="cuda")
            lib = lambda: torch.mm(a, b, out=c_lib)  # noqa
            lib()
            t_o, t_l = [], []
            for _ in range(3):
                t_o.append(ev(ours, 3))
                t_l.append(ev(lib, 3))
            f = 2.0 * n ** 3
            res[variant] = {"tflops": f / min(t_o) / 1e12, "rel_err": err}
            res["cublas_sgemm_tflops"] = f / min(t_l) / 1e12
            del ref
        for v in ("ffma2", "ffma2k32", "ffma2k16j", "ffma2k16"):
            res[v + "_vs_cublas"] = res[v]["tflops"] / res["cublas_sgemm_tflops"]
        print(json.dumps(res), flush=True)
        del a, b, c
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
