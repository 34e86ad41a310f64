#!/bin/bash
# session-4 call j: run-to-run spread of the bench line on the round's final code
# (the paper averages 5 runs): 5 independent runs of the driver's command on cfg 4
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4j
nvidia-smi > gpurun_out/${T}_smi.txt 2>&1
for r in 1 2 3 4 5; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench4_run$r.log 2>&1
  echo "run $r exit $?" >> gpurun_out/${T}_bench4_run$r.log
done
echo done
