#!/usr/bin/env bash
# Two default bench runs (the driver's invocation) plus the reference arm.
set -u
OUT=gpurun_out/${1:-r02_bench2}; mkdir -p $OUT
for i in 1 2; do
  timeout 900 python bench.py > $OUT/bench_$i.json 2> $OUT/bench_$i.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
echo done
