#!/usr/bin/env bash
# (dev) usage: bash tools/group_sustained.sh <tag> -- raster-group sweep of the pair
# kernel (dynamic scheduler, TMA-store epilogue) at 16384^3: ncu DRAM bytes per
# launch, then a sustained interleaved comparison (raster_sweep.py) with cuBLAS.
set -u
OUT=gpurun_out/${1:-gsus}; mkdir -p "$OUT"
M=dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for g in 4 6 8 12 16; do
  POAS_TC_GROUP=$g timeout 300 ncu --metrics $M --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv \
    python tools/ncu_target.py tc 16384 > "$OUT/t.csv" 2>&1
  vals=$(grep -E "dram__bytes_read|gpu__time|cycles_elapsed|tensor" "$OUT/t.csv" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}')
  echo "g$g $vals" >> "$OUT/groups.txt"
done
rm -f "$OUT/t.csv"
timeout 900 python tools/raster_sweep.py --rounds 6 \
  --variants "g4=POAS_TC_GROUP:4;g6=POAS_TC_GROUP:6;g8=POAS_TC_GROUP:8;g12=POAS_TC_GROUP:12;g16=POAS_TC_GROUP:16;cublas=cublas" \
  16384 > "$OUT/sweep.json" 2> "$OUT/sweep.err"
