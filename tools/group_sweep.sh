#!/usr/bin/env bash
# Raster-group sweep of the tensor kernels under the dynamic scheduler:
# ncu DRAM bytes + duration per launch for each (kernel, group, orientation)
# at 16384^3 and 32768^3. Usage (via gpurun): bash tools/group_sweep.sh <tag>
set -u
OUT=gpurun_out/${1:-groups}
mkdir -p "$OUT"
M=dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second
for n in 16384 32768; do
  for v in 2cta 1cta; do
    for g in 2 4 8 16; do
      for r in m n; do
        POAS_TC_KERNEL=$v POAS_TC_GROUP=$g POAS_TC_RASTER=$r timeout 300 ncu --metrics $M \
          --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv python tools/ncu_target.py tc $n \
          > "$OUT/t.csv" 2>&1
        vals=$(grep -E "dram__bytes_read|gpu__time|cycles_elapsed" "$OUT/t.csv" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}')
        echo "$n $v g$g r$r $vals" >> "$OUT/groups.txt"
      done
    done
  done
done
rm -f "$OUT/t.csv"
timeout 900 python tools/raster_sweep.py --rounds 5 16384 32768 > "$OUT/sweep.json" 2> "$OUT/sweep.err"
echo done
