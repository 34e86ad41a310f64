#!/bin/bash
# session-3 final validation: GPU tests, smoke, bench cfg 4 (default) and cfg 5, sharded 1-rank bench (layout
# push), reference arm, launch lists of the bench command (the plan fixed to the one the timed run picks, since
# the set-up timing is distorted under ncu), median-window launch lists, ncu --set full of the top kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${T:-s3q}
nvidia-smi > gpurun_out/${T}_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench4.log 2>&1
echo "bench exit $?" >> gpurun_out/${T}_bench4.log
timeout 1200 python bench.py --config 5 --no-cpu-baseline > gpurun_out/${T}_bench5.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --sharded --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench4_sharded1.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_reference.log 2>&1
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --plan cb"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/${T}_launches4.csv $B > gpurun_out/${T}_ncu_launch4.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_launches4.csv gpurun_out/${T}_launches4.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attr_tile -s 20 -c 1 -o gpurun_out/${T}_tile4 $B > gpurun_out/${T}_ncu_tile4.log 2>&1
B5="python bench.py --config 5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --plan sell"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/${T}_launches5.csv $B5 > gpurun_out/${T}_ncu_launch5.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_launches5.csv gpurun_out/${T}_launches5.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attr_sell_g -s 20 -c 1 -o gpurun_out/${T}_sell5 $B5 > gpurun_out/${T}_ncu_sell5.log 2>&1
for cs in "4 584" "5 584"; do
  set -- $cs
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_median$1.csv python scripts/late_window_launches.py $1 $2 12 stats > gpurun_out/${T}_median$1.log 2>&1
  python scripts/ncu_summary.py launches gpurun_out/${T}_median$1.csv gpurun_out/${T}_median$1.txt
done
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_spread_runs -s 1 -c 1 \
  -o gpurun_out/${T}_runs5 python scripts/late_window_launches.py 5 600 3 stats > gpurun_out/${T}_ncu_runs5.log 2>&1
echo done
