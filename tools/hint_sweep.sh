#!/usr/bin/env bash
# (dev) usage: bash tools/hint_sweep.sh <tag> -- per-operand L2 policy hints of the
# pair kernel's TMA loads at 16384^3 (dynamic scheduler): ncu DRAM bytes per launch.
set -u
OUT=gpurun_out/${1:-hints}; mkdir -p "$OUT"
M=dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for ab in normal:normal last:normal last:first normal:first first:last normal:last; do
  ha=${ab%%:*}; hb=${ab##*:}
  POAS_TC_HINT_A=$ha POAS_TC_HINT_B=$hb timeout 300 ncu --metrics $M --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv \
    python tools/ncu_target.py tc 16384 > "$OUT/t.csv" 2>&1
  vals=$(grep -E "dram__bytes_read|gpu__time|cycles_elapsed|tensor" "$OUT/t.csv" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}')
  echo "A=$ha B=$hb $vals" >> "$OUT/hints.txt"
done
rm -f "$OUT/t.csv"
