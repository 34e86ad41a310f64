cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/tile_timing_probe.py 4 > gpurun_out/r2n_timing.log 2>&1
echo done >> gpurun_out/r2n_timing.log
