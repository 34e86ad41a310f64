TAG=${1:-prof}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_attr_cb.py -m gpu -v --timeout 300 -p no:cacheprovider --durations=0 > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python scripts/attr_probe.py 5 10 > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_attr_csr|k_spmv" -c 2 -o gpurun_out/${TAG}_csr5 python scripts/attr_probe.py 5 10 > gpurun_out/${TAG}_ncu.log 2>&1
