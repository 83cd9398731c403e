#!/usr/bin/env bash
# Epilogue warps of the 256x256 pair tiles: default (8 for one-wave GEMMs,
# else 4) vs the previous tree (4), and forced 8 (POAS_TC_EPI=8).
set -u
OUT=gpurun_out/${1:-r02_epi256b}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_executor.py -m gpu -q -x > $OUT/pytest.txt 2>&1 || { echo "tests failed"; tail -30 $OUT/pytest.txt; exit 1; }
tail -1 $OUT/pytest.txt
S="1536 1792 2048 2560 3072 4096 6144"
for i in 1 2; do
  POAS_SIZES_VARIANTS=default timeout 300 python tools/tc_sizes.py $S > $OUT/sizes_new_$i.json 2>&1
  POAS_TREE=_prev POAS_SIZES_VARIANTS=default timeout 300 python tools/tc_sizes.py $S > $OUT/sizes_prev_$i.json 2>&1
  POAS_TC_EPI=8 POAS_SIZES_VARIANTS=default timeout 300 python tools/tc_sizes.py $S > $OUT/sizes_epi8_$i.json 2>&1
done
