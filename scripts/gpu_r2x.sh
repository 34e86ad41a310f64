#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in base8000 pred base8000 pred; do
  timeout 300 python scripts/tile_variant_probe.py 4 $v >> gpurun_out/r2x_variants.log 2>&1
done
for v in base8000 pred; do timeout 300 python scripts/tile_variant_probe.py 5 $v >> gpurun_out/r2x_variants.log 2>&1; done
