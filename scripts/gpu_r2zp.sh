#!/bin/bash
# ncu evidence for the current kernels: bench launch list (cfg 4), ncu --set full of
# k_attr_tile (cfg 4) and of the field-phase kernels at the median bench window (iteration 584)
T=${1:-r2zp}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/${T}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_ncu_launch.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_launches.csv gpurun_out/${T}_launches.txt
timeout 300 python scripts/attr_tile_probe.py 4 5 > gpurun_out/${T}_tplain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attr_tile -s 2 -c 1 -o gpurun_out/${T}_tile python scripts/attr_tile_probe.py 4 5 > gpurun_out/${T}_ncu_tile.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_spread|k_update|k_row_fwd|k_col|k_row_inv|k_box_count|k_box_scatter|k_box_scan|k_bbox|k_prep" -c 11 \
  -o gpurun_out/${T}_field4 python scripts/late_window_launches.py 4 584 1 > gpurun_out/${T}_field4.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_med_launches4.csv python scripts/late_window_launches.py 4 584 3 > gpurun_out/${T}_med4.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_med_launches4.csv gpurun_out/${T}_med_launches4.txt
cat gpurun_out/${T}_launches.txt gpurun_out/${T}_med_launches4.txt
