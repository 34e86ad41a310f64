#!/bin/bash
# session-3 call f: spread over the recorded box order (auto) vs the sort every iteration; re-sort thresholds
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s3f
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -p no:cacheprovider -k "spread" > gpurun_out/${T}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
for rep in 1 2; do
for st in 300 600 900; do
  for sp in 0 1; do
    timeout 300 python scripts/step_variant_probe.py 5 $st product 50 graph $sp >> gpurun_out/${T}_variants.log 2>&1
    timeout 300 python scripts/step_variant_probe.py 4 $st product 50 graph $sp >> gpurun_out/${T}_variants.log 2>&1
  done
  for v in rs4 rs8 rs32 rs64; do
    timeout 300 python scripts/step_variant_probe.py 5 $st $v 50 graph 0 >> gpurun_out/${T}_variants.log 2>&1
    timeout 300 python scripts/step_variant_probe.py 4 $st $v 50 graph 0 >> gpurun_out/${T}_variants.log 2>&1
  done
done
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches5.csv python scripts/late_window_launches.py 5 600 6 > gpurun_out/${T}_ncu5.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_launches5.csv gpurun_out/${T}_launches5.txt
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches4.csv python scripts/late_window_launches.py 4 600 6 > gpurun_out/${T}_ncu4.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_launches4.csv gpurun_out/${T}_launches4.txt
echo done
