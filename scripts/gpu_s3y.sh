#!/bin/bash
# session-3 call y: the move's field grid through L1 instead of shared memory at N <= 113
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s3y
for rep in 1 2; do
for v in product movel1 moves3600; do
  for cs in "4 300" "4 600" "5 600" "5 900"; do
    set -- $cs
    timeout 300 python scripts/step_variant_probe.py $1 $2 $v 50 graph 0 >> gpurun_out/${T}_variants.log 2>&1
  done
done
done
echo done
