#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in pred sched pred sched; do
  timeout 300 python scripts/tile_variant_probe.py 4 $v >> gpurun_out/r2y_variants.log 2>&1
done
timeout 300 python scripts/attr_tile_probe.py 4 > gpurun_out/r2y_probe4.log 2>&1
timeout 900 python -m pytest tests/test_gpu_attr_cb.py -x -q > gpurun_out/r2y_pytest.log 2>&1
tail -3 gpurun_out/r2y_pytest.log
