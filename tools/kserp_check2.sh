#!/usr/bin/env bash
# (dev) usage: bash tools/kserp_check2.sh <tag> -- K-serpentine at 32768^3 (wave scheduler)
# and 8192^3: ncu DRAM bytes per launch, sustained A/B at 32768^3.
set -u
OUT=gpurun_out/${1:-kserp2}; mkdir -p "$OUT"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for cfg in "32768:0" "32768:1" "8192:0" "8192:1"; do
  n=${cfg%%:*}; ks=${cfg##*:}
  POAS_TC_KSERP=$ks timeout 300 ncu --metrics $M --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv \
    python tools/ncu_target.py tc $n > "$OUT/t.csv" 2>&1
  vals=$(grep -E "dram__bytes|gpu__time|cycles_elapsed|tensor" "$OUT/t.csv" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}')
  echo "n=$n kserp=$ks $vals" >> "$OUT/dram.txt"
done
rm -f "$OUT/t.csv"
cat "$OUT/dram.txt"
AB_N=32768 timeout 900 python tools/ab_env.py "" "POAS_TC_KSERP:1" 4 > "$OUT/ab32768.json" 2>&1
tail -3 "$OUT/ab32768.json"
