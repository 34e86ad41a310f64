TAG=${1:-q}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_quality.py -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python scripts/hypothesis4.py > gpurun_out/${TAG}_h4.log 2>&1
