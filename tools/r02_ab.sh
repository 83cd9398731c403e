#!/usr/bin/env bash
# Round-2 A/B pass: sustained energy per GEMM of the tensor kernel (and knob
# variants) vs cuBLAS at 16384^3, plus one ncu --set full capture of each.
set -u
OUT=gpurun_out/${1:-r02_ab}
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > "$OUT/gpu.txt" 2>&1
POAS_AB_VARIANTS="kserp0:POAS_TC_KSERP=0;g16:POAS_TC_GROUP=16;g4:POAS_TC_GROUP=4;static:POAS_TC_SCHED=static" \
  timeout 600 python tools/energy_ab.py 16384 2.0 3 > "$OUT/energy_16384.json" 2> "$OUT/energy_16384.err"
timeout 300 python tools/energy_ab.py 8192 1.5 3 > "$OUT/energy_8192.json" 2> "$OUT/energy_8192.err"
timeout 600 ncu --set full --clock-control none -k regex:nvjet -s 2 -c 1 -o "$OUT/prof_cublas_16384" \
  python tools/ncu_cublas.py 16384 > "$OUT/ncu_cublas.log" 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_2cta -s 2 -c 1 \
  -o "$OUT/prof_tc_16384" python tools/ncu_target.py tc 16384 > "$OUT/ncu_tc.log" 2>&1
echo done
