#!/bin/bash
# session-4 call g: LPT weight of the tiled plan's panels with a penalty on hub rows (probe builds), cfg 4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4g
bash scripts/tile_variants.sh h32k200 "-DTILE_HUB_MIN=32768 -DTILE_HUB_PM=200" h64k300 "-DTILE_HUB_MIN=65536 -DTILE_HUB_PM=300" \
  h16k150 "-DTILE_HUB_MIN=16384 -DTILE_HUB_PM=150" h48k250 "-DTILE_HUB_MIN=49152 -DTILE_HUB_PM=250" \
  h32k400 "-DTILE_HUB_MIN=32768 -DTILE_HUB_PM=400" > gpurun_out/${T}_build.log 2>&1
for rep in 1 2 3; do
  for v in product h32k200 h64k300 h16k150 h48k250 h32k400; do
    timeout 300 python scripts/tile_variant_probe.py 4 $v >> gpurun_out/${T}_variants.jsonl 2>> gpurun_out/${T}_variants.err
  done
done
echo done
