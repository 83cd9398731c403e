#!/usr/bin/env bash
# Wide pair tile: per-tile MMA/epilogue trace, staging boxes A/B.
set -u
OUT=gpurun_out/${1:-r02_wide2}
mkdir -p "$OUT"
for v in "2cta512:2" "2cta512:4" "2cta:2"; do
  k=${v%%:*}; bx=${v##*:}
  POAS_TC_KERNEL=$k POAS_TC_BOXES=$bx POAS_TC_TRACE=1 timeout 120 python tools/ncu_target.py tc 16384 > "$OUT/trace_${k}_${bx}.txt" 2>&1
done
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "wide" > "$OUT/pytest_wide.txt" 2>&1
POAS_TC_BOXES=4 timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "wide or variants or panels or pitch" > "$OUT/pytest_wide_boxes4.txt" 2>&1
POAS_AB_VARIANTS="boxes4:POAS_TC_BOXES=4" \
  timeout 600 python tools/energy_ab.py 16384 2.0 4 > "$OUT/energy_16384.json" 2> "$OUT/energy_16384.err"
echo done
