TAG=${1:-upd}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "step_parity or ten_iter or runner or edge or ragged or shards" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench.log 2>&1
timeout 600 python bench.py --config 5 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench5.log 2>&1
