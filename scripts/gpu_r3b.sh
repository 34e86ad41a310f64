#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in sortonly loc1024 loc4096; do
  timeout 300 python scripts/step_variant_probe.py 5 600 $v >> gpurun_out/r3b_variants.log 2>&1
  timeout 300 python scripts/step_variant_probe.py 4 990 $v >> gpurun_out/r3b_variants.log 2>&1
  timeout 300 python scripts/step_variant_probe.py 5 100 $v >> gpurun_out/r3b_variants.log 2>&1
  timeout 300 python scripts/step_variant_probe.py 3 990 $v >> gpurun_out/r3b_variants.log 2>&1
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -x -q > gpurun_out/r3b_pytest.log 2>&1
tail -3 gpurun_out/r3b_pytest.log
