TAG=${1:-sellp}; CFG=${2:-5}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TSNET_SELL=${SELL:-2,4} timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attr_sell -s 2 -c 1 -o gpurun_out/${TAG}_top python scripts/attr_probe.py $CFG 5 > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?" >> gpurun_out/${TAG}_ncu.log
