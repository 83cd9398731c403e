#!/usr/bin/env bash
# Tile-scheduler A/B on one GPU box: kernel tests, DRAM bytes per 16384^3
# launch (ncu) for {1cta,2cta} x {dynamic,static}, interleaved sustained
# timing. Usage (via gpurun): bash tools/sched_experiment.sh <tag>
set -u
OUT=gpurun_out/${1:-sched}
mkdir -p "$OUT"
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -5 > "$OUT/pytest_kernels.txt"
for v in 2cta 1cta; do
  for s in dynamic static; do
    POAS_TC_KERNEL=$v POAS_TC_SCHED=$s timeout 300 ncu --metrics \
      dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second \
      --clock-control none -k regex:tc_gemm -s 2 -c 1 --csv python tools/ncu_target.py tc 16384 \
      > "$OUT/ncu_${v}_${s}.csv" 2>&1
  done
done
timeout 900 python tools/raster_sweep.py 16384 32768 > "$OUT/sweep.json" 2> "$OUT/sweep.err"
echo done
