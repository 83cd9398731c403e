#!/usr/bin/env bash
# Alternate the tensor-kernel size sweep over several built trees.
set -u
OUT=gpurun_out/${1:-r02_bisect}; mkdir -p $OUT
shift
for i in 1 2; do
  for t in "$@"; do
    POAS_TREE=$t POAS_SIZES_VARIANTS=default,2cta timeout 300 python tools/tc_sizes.py 2048 3072 4096 > $OUT/$(basename $t)_$i.json 2>$OUT/$(basename $t)_$i.err
  done
done
