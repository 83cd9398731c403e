#!/usr/bin/env bash
# Short-GEMM probes timed as one CUDA graph (the executor's replay mode)
# vs stream launches (POAS_PROBE_GRAPH=1): GPU suite, smoke, the C2/C5
# sweep both ways (alternating), one default bench.
set -u
OUT=gpurun_out/${1:-r02_graph_probe}; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1; tail -1 $OUT/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; tail -1 $OUT/smoke.txt
timeout 900 python tools/sweep.py > $OUT/sweep_graph.json 2> $OUT/sweep_graph.err
POAS_PROBE_GRAPH=1 timeout 900 python tools/sweep.py > $OUT/sweep_stream.json 2> $OUT/sweep_stream.err
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
echo done
