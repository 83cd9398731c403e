#!/usr/bin/env bash
# Round-2 probe pass (dev): CUDA-core kernel vs cuBLAS SGEMM (timing + ncu),
# small tensor GEMMs vs cuBLAS (timing, traces, cuBLAS kernel names).
set -u
OUT=gpurun_out/${1:-r02_probe}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/gpu.txt 2>&1
timeout 300 python tools/simt_check.py 4096 8192 > $OUT/simt_check.json 2> $OUT/simt_check.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:simt_gemm2_kernel -s 1 -c 1 \
  -o $OUT/prof_simt_square python tools/ncu_target.py simt 8192 8192 0 > $OUT/ncu_simt_square.log 2>&1
cat > /tmp/sgemm.py <<'PY'
import torch
torch.backends.cuda.matmul.allow_tf32 = False
n = 8192
a = torch.randn(n, n, device="cuda"); b = torch.randn(n, n, device="cuda"); c = torch.empty(n, n, device="cuda")
for _ in range(3): torch.mm(a, b, out=c)
torch.cuda.synchronize()
PY
timeout 300 ncu --set full --clock-control none -s 2 -c 1 -k regex:'gemm|nvjet|sgemm|cutlass' \
  -o $OUT/prof_cublas_sgemm python /tmp/sgemm.py > $OUT/ncu_cublas_sgemm.log 2>&1
timeout 300 python tools/small_gemm.py 200 > $OUT/small_gemm.json 2> $OUT/small_gemm.err
for n in 1024 2048; do
  timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/ncu_cublas.py $n > $OUT/ncu_cublas_$n.csv 2>&1
  POAS_TC_TRACE=1 timeout 120 python tools/small_gemm.py one $n ours > $OUT/trace_$n.txt 2>&1
done
echo done
