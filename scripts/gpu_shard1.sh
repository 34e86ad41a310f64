TAG=${1:-sh}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shards.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --sharded --no-cpu-baseline --no-e2e --steps 300 > gpurun_out/${TAG}_bench_sharded1.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 300 > gpurun_out/${TAG}_bench.log 2>&1
