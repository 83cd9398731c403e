#!/usr/bin/env bash
# Final HEAD check on one GPU box: the whole GPU suite, smoke, and two
# default bench runs. Outputs under gpurun_out/<tag>/.
set -u
OUT=gpurun_out/${1:-final}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1; tail -1 $OUT/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
for i in 1 2; do
  timeout 900 python bench.py > $OUT/bench_$i.json 2> $OUT/bench_$i.err
  tail -c 300 $OUT/bench_$i.json
done
echo done
