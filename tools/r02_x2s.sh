#!/usr/bin/env bash
# 256-wide B-sharing clusters at small sizes: parity, sizes, energy at 2048.
set -u
OUT=gpurun_out/${1:-r02_x2s}; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x > $OUT/pytest_kernels.txt 2>&1 || { echo "kernel tests failed"; tail -30 $OUT/pytest_kernels.txt; exit 1; }
tail -1 $OUT/pytest_kernels.txt
for i in 1 2; do
POAS_SIZES_VARIANTS=2cta256x2,default timeout 300 python tools/tc_sizes.py 1536 2048 3072 4096 > $OUT/sizes_$i.json 2>$OUT/sizes_$i.err
done
POAS_AB_VARIANTS="x2:POAS_TC_KERNEL=2cta256x2" timeout 300 python tools/energy_ab.py 2048 1.0 3 > "$OUT/energy_2048.json" 2> "$OUT/energy_2048.err"
POAS_AB_VARIANTS="x2:POAS_TC_KERNEL=2cta256x2" timeout 300 python tools/energy_ab.py 4096 1.0 3 > "$OUT/energy_4096.json" 2> "$OUT/energy_4096.err"
