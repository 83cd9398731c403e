#!/usr/bin/env bash
# 8 epilogue warps for the wide tiles vs the previous tree (4 warps).
set -u
OUT=gpurun_out/${1:-r02_epi8}; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x > $OUT/pytest_kernels.txt 2>&1 || { echo "kernel tests failed"; tail -30 $OUT/pytest_kernels.txt; exit 1; }
tail -1 $OUT/pytest_kernels.txt
for t in . _prev; do
  n=$(basename $t); [ "$n" = "." ] && n=new
  POAS_TREE=$t POAS_TC_TRACE=1 timeout 120 python tools/ncu_target.py tc 16384 > $OUT/trace16k_$n.txt 2>&1
  POAS_TREE=$t POAS_TC_TRACE=1 timeout 120 python tools/ncu_target.py tc 8192 > $OUT/trace8k_$n.txt 2>&1
done
for i in 1 2; do
  for t in . _prev; do
    n=$(basename $t); [ "$n" = "." ] && n=new
    POAS_TREE=$t timeout 300 python tools/energy_ab.py 16384 1.5 2 > $OUT/energy16k_${n}_$i.json 2>/dev/null
    POAS_TREE=$t timeout 300 python tools/energy_ab.py 8192 1.0 2 > $OUT/energy8k_${n}_$i.json 2>/dev/null
  done
done
