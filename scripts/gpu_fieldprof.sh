# ncu --set full of the non-SpMV kernels of one cfg-5 bench step
TAG=${1:-fp}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --config 5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"k_box_count|k_update|k_box_scatter|k_bbox|k_spread" -s 300 -c 5 -o gpurun_out/${TAG}_field $B > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?" >> gpurun_out/${TAG}_ncu.log
