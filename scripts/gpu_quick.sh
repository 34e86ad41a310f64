# quick gpurun call: selected GPU tests, bench cfg4 (plan), ncu of one kernel
# usage: bash scripts/gpu_quick.sh TAG "pytest -k expr" [kernel regex] [extra bench args]
TAG=${1:-q}
KEXPR=${2:-attr_cb}
KREGEX=${3:-k_attr_cb}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -k "$KEXPR" > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
B="python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/${TAG}_bench4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s 5 -c 1 -o gpurun_out/${TAG}_top $B > gpurun_out/${TAG}_ncu.log 2>&1
echo done
