#!/bin/bash
# session-4 call l: validation of the product build with the field chain's programmatic dependent launches:
# GPU suite, smoke, bench cfg 4 (driver command) and cfg 5, launch list of the bench command
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4l
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench4.log 2>&1
echo "bench exit $?" >> gpurun_out/${T}_bench4.log
timeout 1200 python bench.py --config 5 --no-cpu-baseline > gpurun_out/${T}_bench5.log 2>&1
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --plan cb"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/${T}_launches4.csv $B > gpurun_out/${T}_ncu_launch4.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_launches4.csv gpurun_out/${T}_launches4.txt
echo done
