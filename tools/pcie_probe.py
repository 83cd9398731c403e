"""PCIe copy-engine efficiency vs contiguous row width (dev tool): 2-D
cudaMemcpy2DAsync H2D and D2H of a fixed byte count with row widths from 1
KB to fully contiguous, alone and with the other direction running
concurrently. Prints JSON (GB/s)."""
import ctypes
import json
import sys

import torch

rt = None
for name in ("libcudart.so", "libcudart.so.12"):
    try:
        rt = ctypes.CDLL(name)
        break
    except OSError:
        pass
if rt is None:
    import glob
    rt = ctypes.CDLL(sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*"))[0])
rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                 ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
H2D, D2H = 1, 2
TOTAL = 256 << 20  # bytes per copy
PITCH = 64 << 10   # source / destination row pitch (bytes): a 16384-wide fp32 row


def copy2d(dst, src, width, kind, stream):
    rows = TOTAL // width
    rc = rt.cudaMemcpy2DAsync(dst, PITCH, src, PITCH, width, rows, kind, stream)
    assert rc == 0, rc


def main():
    rows_max = TOTAL // 1024
    h_src = torch.empty(rows_max * PITCH, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(rows_max * PITCH, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(rows_max * PITCH, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(rows_max * PITCH, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for width in (1024, 2048, 4096, 8192, 16384, 32768, 65536):
        row = {}
        for mode in ("h2d", "d2h", "both"):
            for _ in range(2):
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                torch.cuda.synchronize()
                e0.record(s1)
                if mode in ("h2d", "both"):
                    copy2d(d_a.data_ptr(), h_src.data_ptr(), width, H2D, s1.cuda_stream)
                if mode in ("d2h", "both"):
                    s2.wait_event(e0)
                    copy2d(h_dst.data_ptr(), d_b.data_ptr(), width, D2H, s2.cuda_stream)
                    s1.wait_stream(s2)
                e1.record(s1)
                torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            row[mode] = round(TOTAL / (ms * 1e-3) / 1e9 * (2 if mode == "both" else 1), 2)
        out[width] = row
    print(json.dumps(out, indent=1))




def calls():
    """Many smaller 2-D D2H copies (the overlapped executor's C blocks),
    with and without a stream-wait-value before each, alone and beside a
    stream of H2D copies. GB/s of the D2H stream."""
    import sys
    sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
    from paper_2209_10245_b200 import poas  # noqa: F401  (flag helpers)
    import paper_2209_10245_b200._lib as L
    lib = L.lib
    total = 1 << 30
    pitch = 16384 * 4
    h = torch.empty(total, dtype=torch.uint8).pin_memory()
    d = torch.empty(total, dtype=torch.uint8, device="cuda")
    h2 = torch.empty(total, dtype=torch.uint8).pin_memory()
    d2 = torch.empty(total, dtype=torch.uint8, device="cuda")
    flag = torch.ones(1, dtype=torch.int32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for rows, width in ((1024, 4096), (2048, 8192), (4096, 16384), (2048, 65536), (16384, 65536)):
        nblk = total // (rows * width)
        for waits in (False, True):
            for busy in (False, True):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(s1)
                if busy:
                    s2.wait_event(e0)
                    rc = rt.cudaMemcpy2DAsync(d2.data_ptr(), pitch, h2.data_ptr(), pitch, pitch,
                                              total // pitch, H2D, s2.cuda_stream)
                    assert rc == 0
                for b in range(nblk):
                    if waits:
                        assert lib.poas_b200_wait_flag(flag.data_ptr(), 1, s1.cuda_stream) == 0
                    # blocks tile a 16384-column fp32 matrix: row pitch 64 KB
                    off = (b % (pitch // width)) * width + (b // (pitch // width)) * rows * pitch
                    rc = rt.cudaMemcpy2DAsync(h.data_ptr() + off, pitch, d.data_ptr() + off, pitch, width,
                                              rows, D2H, s1.cuda_stream)
                    assert rc == 0
                e1.record(s1)
                torch.cuda.synchronize()
                out[f"{rows}x{width}B{' wait' if waits else ''}{' +h2d' if busy else ''}"] = round(
                    total / (e0.elapsed_time(e1) * 1e-3) / 1e9, 2)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "calls":
        calls()
    else:
        main()
