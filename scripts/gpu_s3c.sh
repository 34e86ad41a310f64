#!/bin/bash
# session-3 call c: sliced-ELL CTAs per SM x field-stream priority (cfg 5 overlap); conv alternatives probe
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for v in product s3hi s3lo s2hi; do
  timeout 300 python scripts/step_variant_probe.py 5 600 $v 50 >> gpurun_out/s3c_variants.log 2>&1
  timeout 300 python scripts/step_variant_probe.py 5 300 $v 50 >> gpurun_out/s3c_variants.log 2>&1
done
done
timeout 600 python scripts/conv_probe.py 60 108 162 > gpurun_out/s3c_conv.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3c_conv_launches.csv python scripts/conv_probe.py 60 > gpurun_out/s3c_conv_ncu.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/s3c_conv_launches.csv gpurun_out/s3c_conv_launches.txt
echo done
