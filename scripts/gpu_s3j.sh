#!/bin/bash
# session-3 call j: leaner k_spread_runs (straight-line, one-segment butterfly)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${T:-s3j}
for cs in "5 600" "4 600"; do
  set -- $cs
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches$1_$2.csv python scripts/late_window_launches.py $1 $2 12 stats > gpurun_out/${T}_ncu$1_$2.log 2>&1
  python scripts/ncu_summary.py launches gpurun_out/${T}_launches$1_$2.csv gpurun_out/${T}_launches$1_$2.txt
done
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_spread_runs -s 1 -c 1 \
  -o gpurun_out/${T}_runs5 python scripts/late_window_launches.py 5 600 3 stats > gpurun_out/${T}_ncu_runs5.log 2>&1
for st in 600 900; do
  for sp in 0 1; do
    timeout 300 python scripts/step_variant_probe.py 5 $st product 50 graph $sp >> gpurun_out/${T}_variants.log 2>&1
    timeout 300 python scripts/step_variant_probe.py 4 $st product 50 graph $sp >> gpurun_out/${T}_variants.log 2>&1
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 900 -p no:cacheprovider -k "spread or bench_states or ragged or edge or synthetic or trajectory" > gpurun_out/${T}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
echo done
