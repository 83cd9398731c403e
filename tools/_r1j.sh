set -u
OUT=gpurun_out/r1j; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_executor.py -m gpu -q -x 2>&1 | tail -15 > $OUT/pytest_exec.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --save $OUT/bench > $OUT/bench.json 2> $OUT/bench.err
