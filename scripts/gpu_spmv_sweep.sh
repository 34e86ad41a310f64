# SpMV launch-configuration sweep (attr_probe: CSR kernel timed alone)
TAG=${1:-sweep}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { env "$@" timeout 300 python scripts/attr_probe.py $CFG 30 | sed "s/^/$* /" >> gpurun_out/${TAG}_sweep.log 2>&1; }
for CFG in 4 5; do
  run TSNET_SPMV_CPW=4
  run TSNET_SPMV_CPW=2
  run TSNET_SPMV_CPW=8
  run TSNET_SPMV_U=8
  run TSNET_SPMV_U=2
done
