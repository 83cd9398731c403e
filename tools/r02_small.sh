#!/usr/bin/env bash
# (dev) small-GEMM pass: GPU tests, ours vs cuBLAS (PDL on/off), C5 sweep.
set -u
OUT=gpurun_out/${1:-r02_small}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.txt 2>&1
timeout 300 python tools/small_gemm.py 200 > $OUT/small_gemm.json 2> $OUT/small_gemm.err
POAS_TC_PDL=0 timeout 300 python tools/small_gemm.py 200 > $OUT/small_gemm_nopdl.json 2>> $OUT/small_gemm.err
timeout 900 python tools/sweep.py --quick --c5 > $OUT/sweep.json 2> $OUT/sweep.err
echo done
