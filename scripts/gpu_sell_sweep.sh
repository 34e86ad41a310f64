TAG=${1:-sells}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 4,2 4,3 8,2 2,4 2,6; do echo "TSNET_SELL=$c" >> gpurun_out/${TAG}.log; TSNET_SELL=$c timeout 300 python scripts/attr_probe.py 5 20 2>&1 | grep cfg >> gpurun_out/${TAG}.log; done
