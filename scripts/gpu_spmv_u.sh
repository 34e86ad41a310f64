TAG=${1:-su}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in "TSNET_SPMV_U=4" "TSNET_SPMV_U=2" "TSNET_SPMV_U=8" "TSNET_SPMV_U=4 TSNET_SPMV_WAVES=32" "TSNET_SPMV_U=4 TSNET_SPMV_CTAS=4" "TSNET_SPMV_U=8 TSNET_SPMV_CTAS=4"; do echo "$v $(env $v timeout 300 python scripts/attr_probe.py 4 30 2>&1 | grep cfg | sed 's/.*csr \([0-9.]*\) ms.*/\1/')" >> gpurun_out/${TAG}.log; done
