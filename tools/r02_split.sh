#!/usr/bin/env bash
# Last-wave K split of the pair kernel: parity first (the split test alone,
# then every kernel and executor test), then back-to-back launch times with
# the split (default) and without (POAS_TC_SPLIT=0), alternating.
set -u
OUT=gpurun_out/${1:-r02_split}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k last_wave_split > $OUT/pytest_split.txt 2>&1 || { echo "split tests failed"; tail -30 $OUT/pytest_split.txt; exit 1; }
tail -1 $OUT/pytest_split.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_executor.py tests/test_gpu_fullsize.py -m gpu -q -x > $OUT/pytest.txt 2>&1 || { echo "tests failed"; tail -30 $OUT/pytest.txt; exit 1; }
tail -1 $OUT/pytest.txt
S="2560 4096 4608 5120 8192 16384"
for i in 1 2 3; do
  POAS_SIZES_VARIANTS=default timeout 300 python tools/tc_sizes.py $S > $OUT/sizes_split_$i.json 2>&1
  POAS_TC_SPLIT=0 POAS_SIZES_VARIANTS=default timeout 300 python tools/tc_sizes.py $S > $OUT/sizes_nosplit_$i.json 2>&1
done
timeout 600 python tools/sweep.py > $OUT/sweep.json 2> $OUT/sweep.err
echo done
