#!/usr/bin/env bash
# Panel-major consumer: grouped raster over all panels (default) vs panel order.
set -u
OUT=gpurun_out/${1:-r02_panels2}; mkdir -p $OUT
timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_comm.py tests/test_gpu_multirank.py -q -x > $OUT/pytest.txt 2>&1 || { echo "tests failed"; tail -30 $OUT/pytest.txt; exit 1; }
tail -1 $OUT/pytest.txt
for shape in "8192 8192 8192" "16384 16384 16384" "32768 8192 8192"; do
  tag=$(echo $shape | tr ' ' 'x')
  timeout 300 python tools/panels_ab.py $shape > $OUT/raster_$tag.json 2>&1
  POAS_TC_PANEL_ORDER=panel timeout 300 python tools/panels_ab.py $shape > $OUT/panelorder_$tag.json 2>&1
done
