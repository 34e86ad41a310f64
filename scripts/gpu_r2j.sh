# r2j: tiled SpMV v2 (warp-owned rows, carry combine) -- tests + timing + ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/attr_tile_probe.py 1 20 > gpurun_out/r2j_probe1.log 2>&1; echo "probe1 rc=$?" >> gpurun_out/r2j_probe1.log
timeout 900 python -m pytest tests/test_gpu_attr_cb.py -q -x -p no:cacheprovider > gpurun_out/r2j_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2j_pytest.log
timeout 300 python scripts/attr_tile_probe.py 3 50 > gpurun_out/r2j_probe3.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_probe3.log
timeout 300 python scripts/attr_tile_probe.py 4 50 > gpurun_out/r2j_probe4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attr_tile -s 2 -c 1 -o gpurun_out/r2j_tile python scripts/attr_tile_probe.py 4 5 > gpurun_out/r2j_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2j_probe4.log
