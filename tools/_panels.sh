set -u
OUT=gpurun_out/${1:-panels}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "panels" > $OUT/pytest_panels.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_executor.py -q -x -k "panels" >> $OUT/pytest_panels.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x >> $OUT/pytest_panels.txt 2>&1
