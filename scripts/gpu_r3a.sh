#!/bin/bash
# cfg-5 launch list at a mid stage-B window, plus ncu counters for the field-chain kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/late_window_launches.py 5 600 1 > gpurun_out/r3a_plain5.log 2>&1 || exit 1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r3a_launches5.csv python scripts/late_window_launches.py 5 600 3 > gpurun_out/r3a_ncu5.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/r3a_launches5.csv gpurun_out/r3a_launches5.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_update|k_spread|k_box_count|k_box_scatter|k_row_fwd|k_col|k_row_inv|k_bbox" -c 8 \
  -o gpurun_out/r3a_field5 python scripts/late_window_launches.py 5 600 1 > gpurun_out/r3a_full5.log 2>&1
tail -2 gpurun_out/r3a_full5.log
