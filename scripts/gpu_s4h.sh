#!/bin/bash
# session-4 call h: stronger hub penalties in the tiled plan's LPT weight (probe builds), cfg 4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4h
bash scripts/tile_variants.sh h32k400 "-DTILE_HUB_MIN=32768 -DTILE_HUB_PM=400" h32k600 "-DTILE_HUB_MIN=32768 -DTILE_HUB_PM=600" \
  h32k900 "-DTILE_HUB_MIN=32768 -DTILE_HUB_PM=900" h16k500 "-DTILE_HUB_MIN=16384 -DTILE_HUB_PM=500" \
  h64k600 "-DTILE_HUB_MIN=65536 -DTILE_HUB_PM=600" h8k400 "-DTILE_HUB_MIN=8192 -DTILE_HUB_PM=400" > gpurun_out/${T}_build.log 2>&1
for rep in 1 2 3; do
  for v in product h32k400 h32k600 h32k900 h16k500 h64k600 h8k400; do
    timeout 300 python scripts/tile_variant_probe.py 4 $v >> gpurun_out/${T}_variants.jsonl 2>> gpurun_out/${T}_variants.err
  done
done
echo done
