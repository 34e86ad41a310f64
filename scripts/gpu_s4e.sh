#!/bin/bash
# session-4 call e: run pass with the next chunk's loads under the current chunk (RUNS_PIPE) vs product:
# ncu launch lists at the median windows of cfg 4 and 5, then step timings
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4e
SRC=field bash scripts/tile_variants.sh pipe2 "-DRUNS_PIPE=1 -DRUNS_MINB=2" pipe3 "-DRUNS_PIPE=1" min2 "-DRUNS_MINB=2" > gpurun_out/${T}_build.log 2>&1
for v in product pipe2 pipe3 min2; do
  for cs in "5 600" "4 584"; do
    set -- $cs
    PL=$v; [ $v = product ] && PL=
    PROBE_LIB=$PL timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/${T}_${v}_median$1.csv python scripts/late_window_launches.py $1 $2 12 > gpurun_out/${T}_${v}_median$1.log 2>&1
    python scripts/ncu_summary.py launches gpurun_out/${T}_${v}_median$1.csv gpurun_out/${T}_${v}_median$1.txt
  done
done
for rep in 1 2; do
  for v in product pipe2 pipe3; do
    for cs in "5 600" "4 600"; do
      set -- $cs
      timeout 300 python scripts/step_variant_probe.py $1 $2 $v 50 graph 0 >> gpurun_out/${T}_variants.log 2>&1
    done
  done
done
echo done
