set -u
# (dev) usage: bash tools/epi_warps.sh <tag>  -- kernel tests, trace, small/large timings
OUT=gpurun_out/${1:-epi}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_executor.py -q -x > $OUT/pytest.txt 2>&1
for n in 1024 2048; do
  POAS_TC_TRACE=1 timeout 120 python tools/small_gemm.py one $n ours >> $OUT/trace.txt 2>&1
done
timeout 300 python tools/small_gemm.py 50 > $OUT/small_gemm.json 2> $OUT/small_gemm.err
timeout 300 python tools/ncu_target.py micro > $OUT/micro.json 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed
for n in 2048 16384; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:tc_gemm_2cta -s 2 -c 1 --csv \
    python tools/ncu_target.py tc $n > $OUT/ncu_$n.csv 2>&1
done
