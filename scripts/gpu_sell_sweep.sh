TAG=${1:-sells}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in g4,4 g4,4,5 g4,6 g3,4 g2,4,4 g2,6 g4,4; do echo "TSNET_SELL=$c" >> gpurun_out/${TAG}.log; TSNET_SELL=$c timeout 300 python scripts/attr_probe.py ${CFG:-5} 20 2>&1 | grep cfg | sed 's/.*sell slots/sell slots/' >> gpurun_out/${TAG}.log; done
