#!/usr/bin/env bash
# (dev) usage: bash tools/kserp_hints.sh <tag> -- L2 policy hints on top of the K
# serpentine (16384^3 pair kernel): ncu DRAM bytes per launch, then a sustained A/B.
set -u
OUT=gpurun_out/${1:-khints}; mkdir -p "$OUT"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for ab in normal:normal last:normal normal:last last:first; do
  ha=${ab%%:*}; hb=${ab##*:}
  POAS_TC_HINT_A=$ha POAS_TC_HINT_B=$hb timeout 300 ncu --metrics $M --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv \
    python tools/ncu_target.py tc 16384 > "$OUT/t.csv" 2>&1
  vals=$(grep -E "dram__bytes|gpu__time|cycles_elapsed|tensor" "$OUT/t.csv" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}')
  echo "A=$ha B=$hb $vals" >> "$OUT/dram.txt"
done
rm -f "$OUT/t.csv"
cat "$OUT/dram.txt"
timeout 600 python tools/ab_env.py "" "POAS_TC_HINT_A:last" 8 > "$OUT/ab_alast.json" 2>&1
tail -1 "$OUT/ab_alast.json" | head -c 160; echo
