set -u
OUT=gpurun_out/r02_sizes4; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x > $OUT/pytest_kernels.txt 2>&1 || { echo "kernel tests failed"; tail -30 $OUT/pytest_kernels.txt; exit 1; }
for i in 1 2; do
POAS_SIZES_VARIANTS=default,2cta,2cta512 timeout 300 python tools/tc_sizes.py 2048 3072 4096 5120 6144 8192 > $OUT/new_$i.json 2>$OUT/new_$i.err
done
