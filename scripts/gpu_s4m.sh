#!/bin/bash
# session-4 call m: per-kernel launch lists of the final code at cfg 4's median window (iteration 584, N 108),
# its last window (iteration 990, N 162: the FFT passes' second round of CTAs) and cfg 5's median window
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4m
for cs in "4 584" "4 990" "5 584"; do
  set -- $cs
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_cfg$1_it$2.csv python scripts/late_window_launches.py $1 $2 12 stats > gpurun_out/${T}_cfg$1_it$2.log 2>&1
  python scripts/ncu_summary.py launches gpurun_out/${T}_cfg$1_it$2.csv gpurun_out/${T}_cfg$1_it$2.txt
done
echo done
