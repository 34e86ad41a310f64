TAG=${1:-e2ep}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 1 2 4; do echo "cpw_rows $k" >> gpurun_out/${TAG}.log; TSNET_SPMV_CPW_ROWS=$k TSNET_HOST_CHUNKS=8 TSNET_HOST_TRACE=1 timeout 300 python scripts/e2e_probe.py 4 2>&1 | grep -E "trace|cfg" | tail -2 >> gpurun_out/${TAG}.log; done
for c in 4 6 12; do TSNET_HOST_CHUNKS=$c timeout 300 python scripts/e2e_probe.py 4 2>&1 | grep cfg >> gpurun_out/${TAG}.log; done
