set -u
# (dev) usage: bash tools/simt_tiles.sh <tag>  -- writes gpurun_out/<tag>/
OUT=gpurun_out/${1:-simt}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -k "simt" > $OUT/pytest.txt 2>&1
M=gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,smsp__issue_active.avg.pct_of_peak_sustained_active
for tw in 256 128 128x2; do
  POAS_SIMT_TILE=$tw timeout 300 python -c "
import sys; sys.path.insert(0,'tools'); sys.argv=['x']
import ncu_target as t
import json
r={}
for n in (4096, 8192):
    ms=t.simt(n, n, 0, iters=3, warm=2, exclusive=False); r[n]=round(2*n**3/ms/1e9,1)
print(json.dumps(r))" > $OUT/tflops_$tw.json 2>&1
  POAS_SIMT_TILE=$tw timeout 300 ncu --metrics $M --clock-control none -k regex:simt_gemm_kernel -s 1 -c 1 --csv \
    python tools/ncu_target.py simt 8192 8192 0 > $OUT/ncu_$tw.csv 2>&1
done
