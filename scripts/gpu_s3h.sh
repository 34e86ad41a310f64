#!/bin/bash
# session-3 call h: ncu full of k_spread_runs (cfg 5, runs iterations); tile kernel with 19 / 23 consumer warps
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s3h
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_spread_runs -s 1 -c 1 \
  -o gpurun_out/${T}_runs5 python scripts/late_window_launches.py 5 600 3 stats > gpurun_out/${T}_ncu_runs5.log 2>&1
for rep in 1 2; do
  for v in product tw19 tw23; do
    timeout 300 python scripts/tile_variant_probe.py 4 $v >> gpurun_out/${T}_tile.log 2>&1
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 900 -p no:cacheprovider -k "spread" > gpurun_out/${T}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
echo done
