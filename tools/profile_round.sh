#!/usr/bin/env bash
# ncu evidence for the tensor unit: full capture of the default 16384^3
# launch, DRAM bytes of cuBLAS on the same shape (reference point), and the
# 32768^3 DRAM comparison of both kernels. Usage: bash tools/profile_round.sh <tag>
set -u
OUT=gpurun_out/${1:-prof}
mkdir -p "$OUT"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second
timeout 300 ncu --metrics $M --clock-control none -k regex:"nvjet|gemm|Kernel" -s 2 -c 1 --csv \
  python tools/ncu_cublas.py 16384 > "$OUT/ncu_cublas_16384.csv" 2>&1
for v in 2cta 1cta; do
  POAS_TC_KERNEL=$v timeout 300 ncu --metrics $M --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv \
    python tools/ncu_target.py tc 32768 > "$OUT/ncu_${v}_32768.csv" 2>&1
done
timeout 300 ncu --metrics $M --clock-control none -k regex:"nvjet|gemm|Kernel" -s 2 -c 1 --csv \
  python tools/ncu_cublas.py 32768 > "$OUT/ncu_cublas_32768.csv" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 \
  -o "$OUT/prof_tc2_dyn_16384" python tools/ncu_target.py tc 16384 > "$OUT/ncu_full.log" 2>&1
echo done
