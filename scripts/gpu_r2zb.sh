#!/bin/bash
# tile SpMV variants (scripts/tile_variants.sh builds), cfg 4, twice each
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${1:-r2zb}; shift
for rep in 1 2; do
  for v in "$@"; do
    timeout 300 python scripts/tile_variant_probe.py 4 $v >> gpurun_out/${T}_variants.jsonl 2>> gpurun_out/${T}_variants.err
  done
done
cat gpurun_out/${T}_variants.jsonl
