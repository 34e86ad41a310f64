cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attr_cb.py tests/test_gpu_shards.py -q -x -p no:cacheprovider > gpurun_out/r2s_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2s_pytest.log
timeout 300 python scripts/attr_tile_probe.py 3 20 > gpurun_out/r2s_probe3.log 2>&1
timeout 300 python scripts/attr_tile_probe.py 4 50 > gpurun_out/r2s_probe4.log 2>&1
timeout 300 python scripts/attr_tile_probe.py 4 5 > gpurun_out/r2s_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attr_tile -s 2 -c 1 -o gpurun_out/r2s_tile python scripts/attr_tile_probe.py 4 5 > gpurun_out/r2s_ncu.log 2>&1
echo done >> gpurun_out/r2s_probe4.log
