TAG=${1:-cbp}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python scripts/attr_probe.py 4 10 > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_attr_cb -c 1 -o gpurun_out/${TAG}_top python scripts/attr_probe.py 4 10 > gpurun_out/${TAG}_ncu.log 2>&1
