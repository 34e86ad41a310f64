#!/bin/bash
# session-3 call d: spread paths (sort / runs / auto) -- GPU tests, step timing on cfg 5 and 4, launch list; tile no-init variant
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s3d
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 900 -p no:cacheprovider -k "spread or bench_states or ragged or edge or config5 or teacher or trajectory" > gpurun_out/${T}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
timeout 900 python -m pytest tests/test_gpu_shards.py -q -x --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest_shards.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest_shards.log
for rep in 1 2; do
for sp in 0 1 2; do
  timeout 300 python scripts/step_variant_probe.py 5 600 product 50 graph $sp >> gpurun_out/${T}_variants.log 2>&1
  timeout 300 python scripts/step_variant_probe.py 5 300 product 50 graph $sp >> gpurun_out/${T}_variants.log 2>&1
done
timeout 300 python scripts/step_variant_probe.py 4 600 product 50 graph 0 >> gpurun_out/${T}_variants.log 2>&1
timeout 300 python scripts/tile_variant_probe.py 4 product >> gpurun_out/${T}_tile.log 2>&1
timeout 300 python scripts/tile_variant_probe.py 4 noinit >> gpurun_out/${T}_tile.log 2>&1
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches5.csv python scripts/late_window_launches.py 5 600 3 > gpurun_out/${T}_ncu5.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_launches5.csv gpurun_out/${T}_launches5.txt
timeout 1200 python bench.py --config 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench5.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --sharded --no-cpu-baseline --no-e2e --steps 50 > gpurun_out/${T}_bench4_sharded1.log 2>&1
echo done
