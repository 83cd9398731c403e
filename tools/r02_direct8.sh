#!/usr/bin/env bash
# 256x512 tiles: TMA-store epilogue vs 256-bit register stores (direct8).
set -u
OUT=gpurun_out/${1:-r02_direct8}; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x > $OUT/pytest_kernels.txt 2>&1 || { echo "kernel tests failed"; tail -30 $OUT/pytest_kernels.txt; exit 1; }
tail -1 $OUT/pytest_kernels.txt
for e in tma direct8; do
  POAS_TC_EPILOGUE=$e POAS_TC_KERNEL=2cta512 POAS_TC_TRACE=1 timeout 120 python tools/ncu_target.py tc 16384 > $OUT/trace_$e.txt 2>&1
  POAS_TC_EPILOGUE=$e POAS_TC_KERNEL=2cta512 POAS_TC_TRACE=1 timeout 120 python tools/ncu_target.py tc 8192 > $OUT/trace8k_$e.txt 2>&1
done
POAS_AB_VARIANTS="direct8:POAS_TC_EPILOGUE=direct8;w256:POAS_TC_KERNEL=2cta" timeout 600 python tools/energy_ab.py 16384 2.0 3 > "$OUT/energy_16384.json" 2> "$OUT/energy_16384.err"
POAS_AB_VARIANTS="direct8:POAS_TC_EPILOGUE=direct8;w256:POAS_TC_KERNEL=2cta" timeout 300 python tools/energy_ab.py 8192 1.5 3 > "$OUT/energy_8192.json" 2> "$OUT/energy_8192.err"
POAS_TC_EPILOGUE=direct8 timeout 600 ncu --set full --clock-control none -k regex:tc_gemm_2cta -s 2 -c 1 \
  -o "$OUT/prof_direct8_16384" python tools/ncu_target.py tc 16384 > "$OUT/ncu_direct8.log" 2>&1
