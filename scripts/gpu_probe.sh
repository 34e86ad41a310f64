# usage: bash scripts/gpu_probe.sh TAG "pytest -k expr"
TAG=${1:-probe}; KEXPR=${2:-attr_cb}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider -k "$KEXPR" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
for K in v1 v2 v2u4; do for c in 4 5; do TSNET_ATTR_KERNEL=$K timeout 300 python scripts/attr_probe.py $c 30 | sed "s/^/$K /" >> gpurun_out/${TAG}_probe.log 2>&1; done; done
