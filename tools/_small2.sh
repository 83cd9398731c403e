set -u
OUT=gpurun_out/${1:-small}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > $OUT/pytest_kernels.txt 2>&1
timeout 300 python tools/small_gemm.py 50 > $OUT/small_gemm_tma.json 2> $OUT/small_gemm.err
POAS_TC_EPILOGUE=direct timeout 300 python tools/small_gemm.py 50 > $OUT/small_gemm_direct.json 2>> $OUT/small_gemm.err
timeout 300 python tools/ncu_target.py micro > $OUT/micro_tma.json 2>&1
POAS_TC_EPILOGUE=direct timeout 300 python tools/ncu_target.py micro > $OUT/micro_direct.json 2>&1
for n in 2048; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 \
    -o $OUT/prof_tc_$n python tools/small_gemm.py one $n ours > $OUT/ncu_tc_$n.log 2>&1
done
