#!/bin/bash
# session-3 call v: shard / push tests and the sharded 1-rank bench after the bounded peer waits
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s3v
timeout 900 python -m pytest tests/test_gpu_shards.py tests/test_gpu_parity.py -q --timeout 900 -p no:cacheprovider -k "shard or push or one_rank or step" > gpurun_out/${T}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --sharded --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench4_sharded1.log 2>&1
echo done
