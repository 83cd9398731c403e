#!/usr/bin/env bash
# ncu --set full of ours vs cuBLAS at 2048^3 (one launch each, warm).
set -u
OUT=gpurun_out/${1:-r02_ncu2k}; mkdir -p $OUT
timeout 300 ncu --set full --clock-control none -k regex:tc_gemm_2cta -s 3 -c 1 -o $OUT/ours2k python tools/small_gemm.py one 2048 ours > $OUT/ours.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:nvjet -s 3 -c 1 -o $OUT/cublas2k python tools/small_gemm.py one 2048 cublas > $OUT/cublas.log 2>&1
