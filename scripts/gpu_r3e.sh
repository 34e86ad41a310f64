#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python scripts/step_variant_probe.py 5 600 sortonly >> gpurun_out/r3e_variants.log 2>&1
timeout 300 python scripts/step_variant_probe.py 5 600 product >> gpurun_out/r3e_variants.log 2>&1
cat > /tmp/llw.py <<'PY'
import os, sys
sys.argv = [sys.argv[0]] + sys.argv[2:]
from paper_2509_19785_b200 import tsnet as T
T.LIB_PATH = os.path.join(os.getcwd(), "paper_2509_19785_b200/build/variants/libtsnet_sortonly.so")
exec(open("scripts/late_window_launches.py").read())
PY
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r3e_launches5_sort.csv python /tmp/llw.py x 5 600 3 > gpurun_out/r3e_ncu5s.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/r3e_launches5_sort.csv gpurun_out/r3e_launches5_sort.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"k_spread_local|k_box_count" -c 2 \
  -o gpurun_out/r3e_spread python scripts/late_window_launches.py 5 600 1 > gpurun_out/r3e_full.log 2>&1
tail -2 gpurun_out/r3e_full.log
