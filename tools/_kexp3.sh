set -u
OUT=gpurun_out/${1:-kexp}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > $OUT/pytest_kernels.txt 2>&1
for n in 1024 2048; do
  POAS_TC_TRACE=1 timeout 120 python tools/small_gemm.py one $n ours >> $OUT/trace.txt 2>&1
  POAS_TC_EPILOGUE=direct POAS_TC_TRACE=1 timeout 120 python tools/small_gemm.py one $n ours >> $OUT/trace_direct.txt 2>&1
  POAS_TC_EPI_SKIP=1 POAS_TC_TRACE=1 timeout 120 python tools/small_gemm.py one $n ours >> $OUT/trace_skip.txt 2>&1
done
timeout 300 python tools/small_gemm.py 50 > $OUT/small_gemm.json 2> $OUT/small_gemm.err
timeout 300 python tools/ncu_target.py micro > $OUT/micro.json 2>&1
