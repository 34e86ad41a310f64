TAG=${1:-bq}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench4.log 2>&1
timeout 900 python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 200 > gpurun_out/${TAG}_bench5.log 2>&1
pgrep -a nvidia-smi > gpurun_out/${TAG}_leftover.txt 2>&1; echo done
