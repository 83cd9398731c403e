#!/usr/bin/env bash
# Wave-synchronised static scheduler vs dynamic claiming: kernel tests, DRAM
# bytes (ncu) and interleaved sustained timing. Usage: bash tools/wave_experiment.sh <tag>
set -u
OUT=gpurun_out/${1:-wave}
mkdir -p "$OUT"
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > "$OUT/pytest_kernels.txt" 2>&1
M=dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second
for n in 16384 32768; do
  for cfg in "2cta 8 m wave" "2cta 8 m dynamic" "2cta 4 n wave" "1cta 16 m wave" "1cta 16 m dynamic"; do
    set -- $cfg
    POAS_TC_KERNEL=$1 POAS_TC_GROUP=$2 POAS_TC_RASTER=$3 POAS_TC_SCHED=$4 timeout 300 ncu --metrics $M \
      --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv python tools/ncu_target.py tc $n > "$OUT/t.csv" 2>&1
    vals=$(grep -E "dram__bytes_read|gpu__time|cycles_elapsed" "$OUT/t.csv" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}')
    echo "$n $cfg $vals" >> "$OUT/dram.txt"
  done
done
rm -f "$OUT/t.csv"
V="2cta:g8:dyn=POAS_TC_KERNEL:2cta,POAS_TC_GROUP:8;2cta:g8:wave=POAS_TC_KERNEL:2cta,POAS_TC_GROUP:8,POAS_TC_SCHED:wave;2cta:g4n:wave=POAS_TC_KERNEL:2cta,POAS_TC_GROUP:4,POAS_TC_RASTER:n,POAS_TC_SCHED:wave;1cta:g16:dyn=POAS_TC_KERNEL:1cta,POAS_TC_GROUP:16;1cta:g16:wave=POAS_TC_KERNEL:1cta,POAS_TC_GROUP:16,POAS_TC_SCHED:wave;cublas=cublas"
timeout 900 python tools/raster_sweep.py --rounds 5 --variants "$V" 16384 32768 > "$OUT/sweep.json" 2> "$OUT/sweep.err"
echo done
