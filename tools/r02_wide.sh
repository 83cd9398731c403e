#!/usr/bin/env bash
# 256x512 pair tiles: kernel parity tests, sustained energy A/B vs the
# 256x256 tile and cuBLAS, ncu of the wide kernel.
set -u
OUT=gpurun_out/${1:-r02_wide}
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > "$OUT/gpu.txt" 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "wide or variant_choice" > "$OUT/pytest_wide.txt" 2>&1
rc=$?
echo "wide tests rc=$rc" >> "$OUT/pytest_wide.txt"
if [ $rc -ne 0 ]; then echo "wide tests failed"; exit 1; fi
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > "$OUT/pytest_kernels.txt" 2>&1
POAS_AB_VARIANTS="w256:POAS_TC_KERNEL=2cta" \
  timeout 600 python tools/energy_ab.py 16384 2.0 3 > "$OUT/energy_16384.json" 2> "$OUT/energy_16384.err"
POAS_AB_VARIANTS="w256:POAS_TC_KERNEL=2cta" \
  timeout 300 python tools/energy_ab.py 8192 1.5 3 > "$OUT/energy_8192.json" 2> "$OUT/energy_8192.err"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_2cta -s 2 -c 1 \
  -o "$OUT/prof_tc512_16384" python tools/ncu_target.py tc 16384 > "$OUT/ncu_tc.log" 2>&1
echo done
