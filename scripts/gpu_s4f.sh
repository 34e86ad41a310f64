#!/bin/bash
# session-4 call f: per-CTA cycles of the tiled SpMV on cfg 4 (TILE_DIAG=3 probe build)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4f
bash scripts/tile_variants.sh timing "-DTILE_DIAG=3" > gpurun_out/${T}_build.log 2>&1
timeout 300 python scripts/tile_timing_probe.py 4 timing > gpurun_out/${T}_timing4.log 2>&1
echo done
