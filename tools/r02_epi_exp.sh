#!/usr/bin/env bash
# Epilogue drain experiments on the pair kernels (trace slots 10-13).
set -u
OUT=gpurun_out/${1:-r02_epi_exp}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x > $OUT/pytest_kernels.txt 2>&1 || { echo "kernel tests failed"; tail -30 $OUT/pytest_kernels.txt; exit 1; }
for k in 2cta512 2cta; do
  POAS_TC_KERNEL=$k POAS_TC_TRACE=1 timeout 120 python tools/ncu_target.py tc 16384 > $OUT/trace_${k}.txt 2>&1
  POAS_TC_KERNEL=$k POAS_TC_EPI_SKIP=1 POAS_TC_TRACE=1 timeout 120 python tools/ncu_target.py tc 16384 > $OUT/trace_${k}_skip.txt 2>&1
done
POAS_AB_VARIANTS="w256:POAS_TC_KERNEL=2cta" timeout 600 python tools/energy_ab.py 16384 2.0 3 > "$OUT/energy_16384.json" 2> "$OUT/energy_16384.err"
echo done
