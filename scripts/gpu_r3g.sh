#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in product u512v4 u1024v4 product u512v4 u1024v4; do
  timeout 300 python scripts/step_variant_probe.py 5 600 $v >> gpurun_out/r3g_variants.log 2>&1 || exit 1
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r3g_launches5.csv python scripts/late_window_launches.py 5 600 3 > gpurun_out/r3g_ncu5.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/r3g_launches5.csv gpurun_out/r3g_launches5.txt
