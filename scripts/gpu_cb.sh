TAG=${1:-cb}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attr_cb.py tests/test_gpu_shards.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
for c in 4 5 3; do timeout 300 python scripts/attr_probe.py $c 30 >> gpurun_out/${TAG}_probe.log 2>&1; done
