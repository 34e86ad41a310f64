TAG=${1:-cb}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attr_cb.py tests/test_gpu_shards.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
for c in 4 5 3; do timeout 300 python scripts/attr_probe.py $c 30 >> gpurun_out/${TAG}_probe.log 2>&1; done
timeout 300 python scripts/attr_probe.py 4 10 > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attr_cb -c 1 -o gpurun_out/${TAG}_top python scripts/attr_probe.py 4 10 > gpurun_out/${TAG}_ncu.log 2>&1
