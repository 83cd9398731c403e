#!/usr/bin/env bash
# Static-prediction bias at C3/C4: the default probe regime (0.5 s warm-up,
# 20 ms pre-roll) against a longer one, alternating, two runs each.
set -u
OUT=gpurun_out/${1:-r02_probe_regime}; mkdir -p $OUT
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-sweep --no-cpu-baseline > $OUT/default_$i.json 2> $OUT/default_$i.err
  timeout 600 python bench.py --steps 20 --warmup 3 --no-sweep --no-cpu-baseline --probe-warmup 1.5 --preroll 60 > $OUT/long_$i.json 2> $OUT/long_$i.err
done
echo done
