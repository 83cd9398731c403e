set -u
# (dev) usage: bash tools/trace_tc.sh <tag>  -- writes gpurun_out/<tag>/
OUT=gpurun_out/${1:-trace}; mkdir -p $OUT
for n in 1024 2048 4096 8192; do
  POAS_TC_TRACE=1 timeout 120 python tools/small_gemm.py one $n ours >> $OUT/trace.txt 2>&1
done
