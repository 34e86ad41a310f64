#!/bin/bash
# session-3 call s: run-pass occupancy variants (points per lane x CTAs per SM)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s3s
for rep in 1 2; do
for st in 600 900; do
  for v in product rp4m4 rp8m4 rp16m2; do
    timeout 300 python scripts/step_variant_probe.py 5 $st $v 50 graph 0 >> gpurun_out/${T}_variants.log 2>&1
    timeout 300 python scripts/step_variant_probe.py 4 $st $v 50 graph 0 >> gpurun_out/${T}_variants.log 2>&1
  done
done
done
echo done
