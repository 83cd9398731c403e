#!/usr/bin/env bash
# Tensor kernel launch times over square sizes: this tree (and _old, a
# worktree of an earlier commit, when present), alternating.
set -u
OUT=gpurun_out/${1:-r02_sizes}; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x > $OUT/pytest_kernels.txt 2>&1 || { echo "kernel tests failed"; tail -30 $OUT/pytest_kernels.txt; exit 1; }
tail -1 $OUT/pytest_kernels.txt
for i in 1 2; do
  if [ -d _old ]; then
    POAS_TREE=_old POAS_SIZES_VARIANTS=default,2cta timeout 300 python tools/tc_sizes.py 1024 2048 3072 4096 8192 > $OUT/old_$i.json 2>$OUT/old_$i.err
  fi
  timeout 300 python tools/tc_sizes.py 1024 2048 3072 4096 8192 > $OUT/new_$i.json 2>$OUT/new_$i.err
done
POAS_TC_KERNEL=2cta512x2 timeout 60 python -c "
import sys; sys.path.insert(0,'.')
from paper_2209_10245_b200 import poas
print('x2 clusters resident:', poas.lib.poas_b200_tc_kernel_name(16384,16384,16384))" > $OUT/x2_name.txt 2>&1
