# r2b: tiled column-blocked SpMV -- correctness tests + cfg 4 / cfg 3 timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/attr_tile_probe.py 1 20 > gpurun_out/r2b_probe1.log 2>&1; echo "probe1 rc=$?" >> gpurun_out/r2b_probe1.log
timeout 900 python -m pytest tests/test_gpu_attr_cb.py -q -x -p no:cacheprovider > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_pytest.log
timeout 300 python scripts/attr_tile_probe.py 4 50 > gpurun_out/r2b_probe4.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_probe4.log
timeout 300 python scripts/attr_tile_probe.py 3 50 > gpurun_out/r2b_probe3.log 2>&1; echo "rc=$?" >> gpurun_out/r2b_probe3.log
echo done
