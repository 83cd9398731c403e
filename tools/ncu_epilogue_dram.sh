set -u
# (dev) usage: bash tools/ncu_epilogue_dram.sh <tag>  -- writes gpurun_out/<tag>/
OUT=gpurun_out/${1:-dram}; mkdir -p $OUT
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for hc in normal first; do
  for rep in 1 2; do
    POAS_TC_HINT_C=$hc timeout 300 ncu --metrics $M --clock-control none -k regex:tc_gemm_2cta -s 2 -c 1 --csv \
      python tools/ncu_target.py tc 16384 > $OUT/ncu_${hc}_$rep.csv 2>&1
  done
done
POAS_TC_HINT_C=first timeout 300 python tools/ncu_target.py micro > $OUT/micro_first.json 2>&1
timeout 300 python tools/ncu_target.py micro > $OUT/micro_normal.json 2>&1
