#!/usr/bin/env bash
# (dev) usage: bash tools/kserp_check.sh <tag> -- K-serpentine (POAS_TC_KSERP=1):
# parity of every tensor variant, ncu DRAM bytes per 16384^3 launch, sustained A/B.
set -u
OUT=gpurun_out/${1:-kserp}; mkdir -p "$OUT"
POAS_TC_KSERP=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -k "variants or pair or tc" > "$OUT/pytest_kserp.txt" 2>&1
tail -2 "$OUT/pytest_kserp.txt"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for cfg in "2cta:0" "2cta:1" "1cta:0" "1cta:1"; do
  v=${cfg%%:*}; ks=${cfg##*:}
  POAS_TC_KERNEL=$v POAS_TC_KSERP=$ks timeout 300 ncu --metrics $M --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv \
    python tools/ncu_target.py tc 16384 > "$OUT/t.csv" 2>&1
  vals=$(grep -E "dram__bytes|gpu__time|cycles_elapsed|tensor" "$OUT/t.csv" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}')
  echo "kernel=$v kserp=$ks $vals" >> "$OUT/dram.txt"
done
rm -f "$OUT/t.csv"
cat "$OUT/dram.txt"
timeout 600 python tools/ab_env.py "" "POAS_TC_KSERP:1" 8 > "$OUT/ab.json" 2>&1
tail -3 "$OUT/ab.json"
