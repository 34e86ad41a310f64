TAG=${1:-sells}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attr_cb.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "sell" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
for c in g4,4 g8,2 g4,6 g3,4 g6,2; do echo "TSNET_SELL=$c" >> gpurun_out/${TAG}.log; TSNET_SELL=$c timeout 300 python scripts/attr_probe.py ${CFG:-5} 20 2>&1 | grep cfg >> gpurun_out/${TAG}.log; done
