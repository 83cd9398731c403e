#!/usr/bin/env bash
# One GPU-box pass: tests, bench, CLI evaluate, ncu evidence. Outputs under
# gpurun_out/<tag>/. Usage (via gpurun): bash tools/gpu_round.sh <tag> [steps]
set -u
TAG=${1:-round}
STEPS=${2:-20}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > "$OUT/gpu.txt" 2>&1
nproc > "$OUT/host.txt"; lscpu | grep -E "Model name|^CPU\(s\)" >> "$OUT/host.txt"

timeout 900 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.txt" 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.txt" 2>&1
timeout 900 python bench.py --steps "$STEPS" --warmup 3 --save "$OUT/bench" > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 600 python bench.py --m-total 65536 --size 8192 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
  > "$OUT/bench_c4.json" 2> "$OUT/bench_c4.err"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"
timeout 900 paper_2209_10245_b200/bin/poas evaluate \
  --units "gpu0.tc=xpu:dev=0:sms=146:dtype=bf16:elem=2:link=hbm:probe=4096-12288;gpu0.simt=gpu:dev=0:sms=2:exclusive=1:elem=4:link=hbm:probe=512-2048" \
  --profiling probes=9,repetitions=3 --policy best-subset --repeats 5 --adapt 3 --out-dir "$OUT/evaluate" > "$OUT/evaluate.txt" 2>&1
# ncu evidence (single launches; numbers under ncu are never bench values)
timeout 300 ncu --set full --clock-control none --import-source on -k regex:simt_gemm2_kernel -s 1 -c 1 \
  -o "$OUT/prof_simt_square" python tools/ncu_target.py simt 8192 8192 0 > "$OUT/ncu_simt_square.log" 2>&1
timeout 300 ncu --set full --clock-control none -k regex:simt_skinny -s 1 -c 1 \
  -o "$OUT/prof_simt_skinny" python tools/ncu_target.py simt 8 16384 2 > "$OUT/ncu_simt_skinny.log" 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-adapt --profile "$OUT/bench/profile_resident.txt" \
  > "$OUT/ncu_launch.log" 2>&1
# the tensor kernel at the bench size, full set (roofline traffic, pipe utilisation)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_2cta -s 2 -c 1 \
  -o "$OUT/prof_tc_16384" python tools/ncu_target.py tc 16384 > "$OUT/ncu_tc_16384.log" 2>&1
# C5 / C2 sweep
timeout 1200 python tools/sweep.py > "$OUT/sweep.json" 2> "$OUT/sweep.err"
echo done
