TAG=${1:-fork}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "runner or step_parity or ten_iter or shards or synthetic" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_smoke.log
B="python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/${TAG}_bench_fork.log 2>&1
TSNET_FIELD_STREAM=0 timeout 600 $B > gpurun_out/${TAG}_bench_nofork.log 2>&1
timeout 600 $B --config 5 > gpurun_out/${TAG}_bench5_fork.log 2>&1
TSNET_FIELD_STREAM=0 timeout 600 $B --config 5 > gpurun_out/${TAG}_bench5_nofork.log 2>&1
