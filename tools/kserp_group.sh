#!/usr/bin/env bash
# (dev) usage: bash tools/kserp_group.sh <tag> -- raster group of the pair kernel
# with the K serpentine at 16384^3: ncu DRAM bytes per launch + sustained A/B vs group 8.
set -u
OUT=gpurun_out/${1:-kgroup}; mkdir -p "$OUT"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for g in 4 6 8 10 12 16; do
  POAS_TC_GROUP=$g timeout 300 ncu --metrics $M --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv \
    python tools/ncu_target.py tc 16384 > "$OUT/t.csv" 2>&1
  vals=$(grep -E "dram__bytes|gpu__time|cycles_elapsed|tensor" "$OUT/t.csv" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}')
  echo "group=$g $vals" >> "$OUT/dram.txt"
done
rm -f "$OUT/t.csv"
cat "$OUT/dram.txt"
for g in 6 12 16; do
  timeout 600 python tools/ab_env.py "POAS_TC_GROUP:8" "POAS_TC_GROUP:$g" 6 > "$OUT/ab_g$g.json" 2>&1
  tail -1 "$OUT/ab_g$g.json" | head -c 200; echo
done
