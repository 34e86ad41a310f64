#!/bin/bash
# round 2, session 2 baseline at HEAD: GPU tests, smoke, bench cfg 4 / 5, launch list,
# ncu full of the SpMV (cfg 4) and of the field-phase kernels (late stage B, cfg 4 and 5)
T=${1:-r2za}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${T}_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench4.log 2> gpurun_out/${T}_bench4.err
timeout 900 python bench.py --config 5 --no-cpu-baseline > gpurun_out/${T}_bench5.log 2> gpurun_out/${T}_bench5.err
timeout 600 python scripts/late_window_launches.py 4 990 3 > gpurun_out/${T}_late4_plain.log 2>&1 && \
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches4.csv python scripts/late_window_launches.py 4 990 3 > gpurun_out/${T}_ncu4.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches5.csv python scripts/late_window_launches.py 5 600 3 > gpurun_out/${T}_ncu5.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_attr_tile|k_spread|k_update|k_row_fwd|k_col|k_row_inv|k_box_count|k_box_scatter|k_bbox" -c 10 \
  -o gpurun_out/${T}_full4 python scripts/late_window_launches.py 4 990 1 > gpurun_out/${T}_full4.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"k_attr_sell_g|k_spread|k_update|k_col|k_box_count|k_box_scatter" -c 7 \
  -o gpurun_out/${T}_full5 python scripts/late_window_launches.py 5 600 1 > gpurun_out/${T}_full5.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_launches4.csv gpurun_out/${T}_launches4.txt
python scripts/ncu_summary.py launches gpurun_out/${T}_launches5.csv gpurun_out/${T}_launches5.txt
tail -3 gpurun_out/${T}_pytest_gpu.log; cat gpurun_out/${T}_bench4.log gpurun_out/${T}_bench5.log | cut -c1-600
