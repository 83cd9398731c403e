#!/usr/bin/env bash
# B-sharing clusters (two CTA pairs, multicast B): parity first, then energy A/B.
set -u
OUT=gpurun_out/${1:-r02_x2}; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > "$OUT/gpu.txt" 2>&1
POAS_TC_KERNEL=2cta512x2 timeout 120 python -c "
import torch,sys
sys.path.insert(0,'.')
from paper_2209_10245_b200 import poas
import oracle
m,n,k=1024,1024,256
A,B=oracle.fill_uniform(m,k,1),oracle.fill_uniform(k,n,2)
a=torch.from_numpy(A).cuda().bfloat16(); b=torch.from_numpy(B).cuda().bfloat16()
c=torch.full((m,n),float('nan'),device='cuda')
poas.tc_gemm(2,m,n,k,a.data_ptr(),k,b.data_ptr(),n,c.data_ptr(),n,num_ctas=8)
torch.cuda.synchronize()
print('first x2 launch rel err', oracle.rel_frobenius(c.cpu().numpy(), oracle.gemm_rows_f64(A,B,2)))
" > $OUT/first.txt 2>&1
echo "first rc=$?" >> $OUT/first.txt
cat $OUT/first.txt
grep -q "rel err" $OUT/first.txt || exit 1
timeout 400 python -m pytest tests/test_gpu_kernels.py -q -x > $OUT/pytest_kernels.txt 2>&1 || { echo "kernel tests failed"; tail -40 $OUT/pytest_kernels.txt; exit 1; }
tail -2 $OUT/pytest_kernels.txt
POAS_TC_KERNEL=2cta512x2 POAS_TC_TRACE=1 timeout 120 python tools/ncu_target.py tc 16384 > $OUT/trace_x2.txt 2>&1
POAS_AB_VARIANTS="x2:POAS_TC_KERNEL=2cta512x2;x2g8:POAS_TC_KERNEL=2cta512x2,POAS_TC_GROUP=8" timeout 600 python tools/energy_ab.py 16384 2.0 3 > "$OUT/energy_16384.json" 2> "$OUT/energy_16384.err"
POAS_AB_VARIANTS="x2:POAS_TC_KERNEL=2cta512x2" timeout 300 python tools/energy_ab.py 8192 1.5 3 > "$OUT/energy_8192.json" 2> "$OUT/energy_8192.err"
POAS_TC_KERNEL=2cta512x2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_2cta -s 2 -c 1 \
  -o "$OUT/prof_x2_16384" python tools/ncu_target.py tc 16384 > "$OUT/ncu_x2.log" 2>&1
echo done
