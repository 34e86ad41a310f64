# SpMV launch-configuration sweep (attr_probe: CSR kernel timed alone)
TAG=${1:-sweep}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
run() { env "$@" timeout 300 python scripts/attr_probe.py $CFG 30 | sed "s/^/$* /" >> gpurun_out/${TAG}_sweep.log 2>&1; }
for CFG in 4 5; do
  run TSNET_SPMV_CPW=3
  run TSNET_SPMV_CPW=1
  run TSNET_SPMV_CPW=2
  run TSNET_SPMV_CPW=6
  run TSNET_SPMV_CTAS=3
  run TSNET_SPMV_CTAS=5
  run TSNET_SPMV_U=8 TSNET_SPMV_CTAS=3
done
