#!/bin/bash
# session-4 call c: source-level ncu of the run pass (k_spread_runs) at cfg 5's median window (runs path)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4c
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_spread_runs -s 1 -c 1 \
  -o gpurun_out/${T}_runs5 python scripts/late_window_launches.py 5 600 3 stats > gpurun_out/${T}_ncu_runs5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_spread_runs -s 1 -c 1 \
  -o gpurun_out/${T}_runs4 python scripts/late_window_launches.py 4 584 3 stats > gpurun_out/${T}_ncu_runs4.log 2>&1
echo done
