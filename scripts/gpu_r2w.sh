#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in o7168 n7680 n7936 n8000 n8048 o7168 n7680 n7936 n8000 n8048; do
  timeout 300 python scripts/tile_variant_probe.py 4 $v >> gpurun_out/r2w_variants.log 2>&1
done
for v in o7168 n7680 n8048; do
  timeout 300 python scripts/tile_variant_probe.py 5 $v >> gpurun_out/r2w_variants.log 2>&1
  timeout 300 python scripts/tile_variant_probe.py 3 $v >> gpurun_out/r2w_variants.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_attr_cb.py -x -q > gpurun_out/r2w_pytest.log 2>&1
tail -3 gpurun_out/r2w_pytest.log
