#!/bin/bash
# session-4 call d: chained steps (a0 from the previous move's bounding box): GPU suite, smoke, bench cfg 4 / 5,
# median-window launch lists
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4d
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench4.log 2>&1
echo "bench exit $?" >> gpurun_out/${T}_bench4.log
timeout 1200 python bench.py --config 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench5.log 2>&1
for cs in "4 584" "5 584"; do
  set -- $cs
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_median$1.csv python scripts/late_window_launches.py $1 $2 12 stats > gpurun_out/${T}_median$1.log 2>&1
  python scripts/ncu_summary.py launches gpurun_out/${T}_median$1.csv gpurun_out/${T}_median$1.txt
done
echo done
