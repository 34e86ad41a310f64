TAG=${1:-p5}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/attr_probe.py 5 10 > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv2 -c 1 -o gpurun_out/${TAG}_spmv5 python scripts/attr_probe.py 5 10 > gpurun_out/${TAG}_ncu.log 2>&1
