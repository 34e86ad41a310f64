#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in sortonly product sortonly product; do
  timeout 300 python scripts/step_variant_probe.py 5 600 $v >> gpurun_out/r3d_variants.log 2>&1
  timeout 300 python scripts/step_variant_probe.py 5 100 $v >> gpurun_out/r3d_variants.log 2>&1
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r3d_launches5.csv python scripts/late_window_launches.py 5 600 3 > gpurun_out/r3d_ncu5.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/r3d_launches5.csv gpurun_out/r3d_launches5.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -x -q > gpurun_out/r3d_pytest.log 2>&1
tail -3 gpurun_out/r3d_pytest.log
