#!/bin/bash
# session-4 call b: packed 112-byte box records of the field grid (7 vector loads per point in the move):
# GPU suite, smoke, ncu of the move at the median windows of cfg 4 and 5, default bench
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4b
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${T}_smoke.log
for cs in "4 584" "5 600"; do
  set -- $cs
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_update -s 2 -c 2 \
    -o gpurun_out/${T}_move$1 python scripts/late_window_launches.py $1 $2 3 > gpurun_out/${T}_ncu_move$1.log 2>&1
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench4.log 2>&1
echo "bench exit $?" >> gpurun_out/${T}_bench4.log
timeout 1200 python bench.py --config 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench5.log 2>&1
echo done
