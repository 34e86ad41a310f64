#!/bin/bash
# session-4 call i: validation of the session's code (packed box records, hub-weighted panel deal):
# GPU suite, smoke, bench cfg 4 (driver defaults) and cfg 5, reference arm, launch list of the bench command,
# ncu --set full of k_attr_tile, per-CTA cycles after the hub penalty
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4i
nvidia-smi > gpurun_out/${T}_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench4.log 2>&1
echo "bench exit $?" >> gpurun_out/${T}_bench4.log
timeout 1200 python bench.py --config 5 --no-cpu-baseline > gpurun_out/${T}_bench5.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_reference.log 2>&1
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --plan cb"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/${T}_launches4.csv $B > gpurun_out/${T}_ncu_launch4.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_launches4.csv gpurun_out/${T}_launches4.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attr_tile -s 20 -c 1 -o gpurun_out/${T}_tile4 $B > gpurun_out/${T}_ncu_tile4.log 2>&1
bash scripts/tile_variants.sh timing "-DTILE_DIAG=3" > gpurun_out/${T}_build.log 2>&1
timeout 300 python scripts/tile_timing_probe.py 4 timing > gpurun_out/${T}_timing4.log 2>&1
echo done
