#!/usr/bin/env bash
# C-store L2 policy (evict_first default vs normal): drain traces and sizes.
set -u
OUT=gpurun_out/${1:-r02_hintc}; mkdir -p $OUT
for h in first normal; do
  POAS_TC_HINT_C=$h POAS_TC_TRACE=1 timeout 120 python tools/ncu_target.py tc 2048 > $OUT/trace2k_$h.txt 2>&1
  POAS_TC_HINT_C=$h POAS_TC_TRACE=1 timeout 120 python tools/ncu_target.py tc 16384 > $OUT/trace16k_$h.txt 2>&1
done
POAS_AB_VARIANTS="hcnormal:POAS_TC_HINT_C=normal" timeout 600 python tools/energy_ab.py 16384 1.5 3 > $OUT/energy_16384.json 2> $OUT/energy_16384.err
POAS_AB_VARIANTS="hcnormal:POAS_TC_HINT_C=normal" timeout 600 python tools/energy_ab.py 2048 0.5 3 > $OUT/energy_2048.json 2> $OUT/energy_2048.err
