#!/bin/bash
# session-3 call o: box_axis, run pass at 3 CTAs/SM, bbox at 4 CTAs/SM -- launch lists and step times
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${T:-s3p}
for cs in "5 600" "4 600"; do
  set -- $cs
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches$1_$2.csv python scripts/late_window_launches.py $1 $2 12 stats > gpurun_out/${T}_ncu$1_$2.log 2>&1
  python scripts/ncu_summary.py launches gpurun_out/${T}_launches$1_$2.csv gpurun_out/${T}_launches$1_$2.txt
done
for rep in 1 2; do
for st in 300 600 900; do
  for sp in 0 1; do
    timeout 300 python scripts/step_variant_probe.py 5 $st product 50 graph $sp >> gpurun_out/${T}_variants.log 2>&1
    timeout 300 python scripts/step_variant_probe.py 4 $st product 50 graph $sp >> gpurun_out/${T}_variants.log 2>&1
  done
done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -q --timeout 900 -p no:cacheprovider -x > gpurun_out/${T}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
echo done
