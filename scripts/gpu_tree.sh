TAG=${1:-tr}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tree.py -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python scripts/tree_probe.py 4 >> gpurun_out/${TAG}_probe.log 2>&1
timeout 600 python scripts/tree_probe.py 3 >> gpurun_out/${TAG}_probe.log 2>&1
