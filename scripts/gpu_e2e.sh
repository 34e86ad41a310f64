# gpurun call: host-step tests + bench e2e for several row-chunk counts
# usage: bash scripts/gpu_e2e.sh TAG
TAG=${1:-e2e}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "step_host or step_parity" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
for c in 1 4 8 16; do
  TSNET_HOST_CHUNKS=$c timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_c$c.log 2>&1
done
