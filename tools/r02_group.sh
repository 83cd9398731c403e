#!/usr/bin/env bash
# Raster group for the 256x512 tiles: sustained A/B at 16384^3 and 8192^3.
set -u
OUT=gpurun_out/${1:-r02_group}; mkdir -p $OUT
POAS_AB_VARIANTS="g4:POAS_TC_GROUP=4;g6:POAS_TC_GROUP=6;g12:POAS_TC_GROUP=12;g16:POAS_TC_GROUP=16" \
  timeout 900 python tools/energy_ab.py 16384 1.5 3 > "$OUT/energy_16384.json" 2> "$OUT/energy_16384.err"
POAS_AB_VARIANTS="g4:POAS_TC_GROUP=4;g6:POAS_TC_GROUP=6;g12:POAS_TC_GROUP=12;g16:POAS_TC_GROUP=16" \
  timeout 600 python tools/energy_ab.py 8192 1.0 3 > "$OUT/energy_8192.json" 2> "$OUT/energy_8192.err"
for g in 4 8 16; do
  POAS_TC_GROUP=$g timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:tc_gemm_2cta -s 2 -c 1 --csv \
    python tools/ncu_target.py tc 16384 > "$OUT/ncu_dram_g$g.csv" 2>&1
done
