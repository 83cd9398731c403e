set -u
OUT=gpurun_out/${1:-small}; mkdir -p $OUT
timeout 300 python tools/small_gemm.py 50 > $OUT/small_gemm.json 2> $OUT/small_gemm.err
for n in 1024 2048; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 3 -c 1 \
    -o $OUT/prof_tc_$n python tools/small_gemm.py one $n ours > $OUT/ncu_tc_$n.log 2>&1
  timeout 300 ncu --set full --clock-control none -k regex:"nvjet|gemm|Kernel" -s 3 -c 1 \
    -o $OUT/prof_cublas_$n python tools/small_gemm.py one $n cublas > $OUT/ncu_cublas_$n.log 2>&1
done
