#!/usr/bin/env bash
# (dev) usage: bash tools/small_variants.sh <tag> -- kernel tests, then small-size timings
# and ncu durations of the pair kernel vs the 128 x 128 single-SM kernel.
set -u
OUT=gpurun_out/${1:-smallv}; mkdir -p "$OUT"
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_executor.py -q -x > "$OUT/pytest.txt" 2>&1
for v in 2cta 1cta128; do
  POAS_TC_KERNEL=$v timeout 300 python tools/small_gemm.py 50 > "$OUT/small_$v.json" 2> /dev/null
  for n in 1024 2048 3072; do
    POAS_TC_KERNEL=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_gemm -s 3 -c 1 --csv \
      python tools/small_gemm.py one $n ours > "$OUT/t.csv" 2>&1
    echo "$v $n $(grep tc_gemm "$OUT/t.csv" | awk -F'","' '{gsub(/"/,"",$NF); print $NF}')" >> "$OUT/ncu.txt"
  done
done
rm -f "$OUT/t.csv"
