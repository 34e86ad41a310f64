#!/bin/bash
# session-3 call a: state at HEAD: GPU tests, smoke, default bench, cfg-5 bench + launch list
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s3a
nvidia-smi > gpurun_out/${T}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench4.log 2>&1
echo "bench exit $?" >> gpurun_out/${T}_bench4.log
timeout 1200 python bench.py --config 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench5.log 2>&1
echo "bench5 exit $?" >> gpurun_out/${T}_bench5.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches5.csv python scripts/late_window_launches.py 5 600 3 > gpurun_out/${T}_ncu5.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_launches5.csv gpurun_out/${T}_launches5.txt
echo done
