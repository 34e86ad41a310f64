# warm-cache launch lists (ncu --cache-control none) of the bench step, cfg 4 and 5
TAG=${1:-wl}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in 4 5; do
B="python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -s 3000 -c 200 --csv --log-file gpurun_out/${TAG}_warm$cfg.csv $B > gpurun_out/${TAG}_ncu$cfg.log 2>&1
done
