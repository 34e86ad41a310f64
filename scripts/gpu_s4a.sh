#!/bin/bash
# session-4 call a: default bench (HEAD), ncu --set full of the move (both variants) and the run pass at the
# median window of cfg 4 and cfg 5
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4a
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench4.log 2>&1
echo "bench exit $?" >> gpurun_out/${T}_bench4.log
for cs in "4 584" "5 600"; do
  set -- $cs
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_update -s 2 -c 2 \
    -o gpurun_out/${T}_move$1 python scripts/late_window_launches.py $1 $2 3 > gpurun_out/${T}_ncu_move$1.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_bbox -s 1 -c 1 \
    -o gpurun_out/${T}_bbox$1 python scripts/late_window_launches.py $1 $2 3 > gpurun_out/${T}_ncu_bbox$1.log 2>&1
done
echo done
