#!/bin/bash
# session-3 call e: FFT pass thread counts / CTAs per SM (cfg 4 median and late windows, cfg 3 late, cfg 5)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s3e
for rep in 1 2; do
for v in product fft256 fftc256 fft384; do
  timeout 300 python scripts/step_variant_probe.py 4 600 $v 50 >> gpurun_out/${T}_variants.log 2>&1
  timeout 300 python scripts/step_variant_probe.py 4 990 $v 50 >> gpurun_out/${T}_variants.log 2>&1
  timeout 300 python scripts/step_variant_probe.py 3 990 $v 50 >> gpurun_out/${T}_variants.log 2>&1
done
done
echo done
for rep in 1 2; do
  timeout 300 python scripts/tile_variant_probe.py 4 product >> gpurun_out/${T}_tile.log 2>&1
  timeout 300 python scripts/tile_variant_probe.py 4 noinit >> gpurun_out/${T}_tile.log 2>&1
done
