TAG=${1:-pm}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pmds.py -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
for c in 4 5 3; do timeout 600 python scripts/pmds_probe.py $c 250 >> gpurun_out/${TAG}_probe.log 2>&1; done
