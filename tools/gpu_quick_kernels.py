"""Quick GPU check of the raw unit kernels against torch fp32 (dev tool)."""
import ctypes as C
import sys
import time

import torch

lib = C.CDLL("paper_2209_10245_b200/libpoas_b200.so")
i64, vp = C.c_int64, C.c_void_p
lib.poas_b200_tc_gemm.argtypes = [C.c_int, i64, i64, i64, vp, i64, vp, i64, vp, i64, C.c_int, C.c_int, vp]
lib.poas_b200_simt_gemm.argtypes = [i64, i64, i64, vp, i64, vp, i64, vp, i64, C.c_int, C.c_int, C.c_int, vp]
lib.poas_b200_last_error.restype = C.c_char_p


def chk(rc):
    if rc != 0:
        raise RuntimeError(f"rc={rc}: {lib.poas_b200_last_error().decode()}")


def rel(c, ref):
    return ((c.double() - ref).norm() / ref.norm()).item()


def tc(M, N, K, dtype=torch.bfloat16, acc=False, ctas=0):
    lda, ldb = (K + 7) // 8 * 8, (N + 7) // 8 * 8
    a = (torch.rand(M, lda, device="cuda") * 2 - 1).to(dtype)[:, :K]
    b = (torch.rand(K, ldb, device="cuda") * 2 - 1).to(dtype)[:, :N]
    c = torch.randn(M, N, device="cuda") if acc else torch.empty(M, N, device="cuda")
    c0 = c.clone()
    d = 2 if dtype == torch.bfloat16 else 1
    chk(lib.poas_b200_tc_gemm(d, M, N, K, a.data_ptr(), lda, b.data_ptr(), ldb, c.data_ptr(), N,
                              int(acc), ctas, None))
    torch.cuda.synchronize()
    ref = a.double() @ b.double() + (c0.double() if acc else 0)
    return rel(c, ref)


def simt(M, N, K, acc=False, ctas=0):
    a = torch.rand(M, K, device="cuda") * 2 - 1
    b = torch.rand(K, N, device="cuda") * 2 - 1
    c = torch.randn(M, N, device="cuda") if acc else torch.empty(M, N, device="cuda")
    c0 = c.clone()
    chk(lib.poas_b200_simt_gemm(M, N, K, a.data_ptr(), K, b.data_ptr(), N, c.data_ptr(), N,
                                int(acc), ctas, 0, None))
    torch.cuda.synchronize()
    ref = a.double() @ b.double() + (c0.double() if acc else 0)
    return rel(c, ref)


def bench_tc(n, iters=10, ctas=0):
    a = torch.randn(n, n, device="cuda").bfloat16()
    b = torch.randn(n, n, device="cuda").bfloat16()
    c = torch.empty(n, n, device="cuda")
    for _ in range(3):
        chk(lib.poas_b200_tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, 0, ctas, None))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        lib.poas_b200_tc_gemm(2, n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, 0, ctas, None)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    # cuBLAS timing comparison
    for _ in range(3):
        torch.matmul(a, b)
    e0.record()
    for _ in range(iters):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms_cublas = e0.elapsed_time(e1) / iters
    return 2 * n**3 / ms / 1e9, 2 * n**3 / ms_cublas / 1e9


def bench_simt(n, iters=5):
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    c = torch.empty(n, n, device="cuda")
    chk(lib.poas_b200_simt_gemm(n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, 0, 0, 0, None))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        lib.poas_b200_simt_gemm(n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, 0, 0, 0, None)
    e1.record()
    torch.cuda.synchronize()
    return 2 * n**3 / (e0.elapsed_time(e1) / iters) / 1e9


if __name__ == "__main__":
    print(torch.cuda.get_device_name(), flush=True)
    for shape in [(128, 256, 64), (256, 512, 128), (1000, 1000, 1000), (129, 300, 72), (2048, 2048, 2048),
                  (64, 4096, 512), (4096, 64, 1024), (3000, 3000, 3000)]:
        print("tc bf16", shape, tc(*shape), flush=True)
    print("tc f16", tc(512, 512, 512, torch.float16), flush=True)
    print("tc acc", tc(640, 768, 320, acc=True), flush=True)
    print("tc 8ctas", tc(1024, 1024, 512, ctas=8), flush=True)
    for shape in [(128, 128, 16), (1000, 1000, 1000), (129, 300, 72), (2048, 2048, 2048), (77, 33, 5)]:
        print("simt", shape, simt(*shape), flush=True)
    print("simt acc", simt(640, 768, 320, acc=True), flush=True)
    for n in [4096, 8192, 16384]:
        print("tc TFLOP/s (ours, cublas)", n, bench_tc(n), flush=True)
    print("tc 16384 on 144 ctas", bench_tc(16384, ctas=144), flush=True)
    for n in [4096, 8192]:
        print("simt TFLOP/s", n, bench_simt(n), flush=True)
