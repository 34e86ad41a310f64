# r2c: ncu of the tiled SpMV on cfg 4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/attr_tile_probe.py 4 5 > gpurun_out/r2c_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attr_tile -s 2 -c 1 -o gpurun_out/r2c_tile python scripts/attr_tile_probe.py 4 5 > gpurun_out/r2c_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2c_ncu.log
