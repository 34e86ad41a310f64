#!/bin/bash
# session-3 call b: field-stream priority / SpMV order probes (cfg 5 sliced ELL, cfg 4 tiled), graph and eager
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for rep in 1 2; do
for v in product prio1 prio1first first; do
  for m in graph eager; do
    timeout 300 python scripts/step_variant_probe.py 5 600 $v 50 $m >> gpurun_out/s3b_variants.log 2>&1
    timeout 300 python scripts/step_variant_probe.py 4 600 $v 50 $m >> gpurun_out/s3b_variants.log 2>&1
  done
done
done
echo done
