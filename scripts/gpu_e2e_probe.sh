TAG=${1:-e2ep}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "step_host" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
TSNET_HOST_CHUNKS=8 TSNET_HOST_TRACE=1 timeout 300 python scripts/e2e_probe.py 4 2>&1 | grep -E "^trace" | tail -1 > gpurun_out/${TAG}.log
for c in 4 6 8 12; do TSNET_HOST_CHUNKS=$c timeout 300 python scripts/e2e_probe.py 4 2>&1 | grep "^cfg" | sed 's/H2D.*device step/device step/' >> gpurun_out/${TAG}.log; done
for c in 4 8; do echo "bench chunks=$c $(TSNET_HOST_CHUNKS=$c timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["e2e"]["value"])')" >> gpurun_out/${TAG}.log; done
