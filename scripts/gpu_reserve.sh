TAG=${1:-res}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for R in 0 2 4 6; do TSNET_SPMV_RESERVE_SMS=$R timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e | sed "s/^/R=$R /" >> gpurun_out/${TAG}_bench.log 2>&1; done
for R in 0 2 4; do TSNET_SPMV_RESERVE_SMS=$R timeout 600 python bench.py --config 5 --steps 200 --warmup 10 --no-cpu-baseline --no-e2e | sed "s/^/R=$R cfg5 /" >> gpurun_out/${TAG}_bench.log 2>&1; done
