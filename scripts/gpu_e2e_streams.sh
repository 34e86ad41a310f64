TAG=${1:-e2es}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider -k "step_host" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
for v in "TSNET_HOST_SPMV_STREAMS=2" "TSNET_HOST_SPMV_STREAMS=1" "TSNET_HOST_SPMV_STREAMS=2" "TSNET_HOST_SPMV_STREAMS=1"; do echo "$v $(env $v timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["e2e"]["value"],1))')" >> gpurun_out/${TAG}.log; done
timeout 1500 python scripts/scaling_variants.py > gpurun_out/${TAG}_scaling.log 2>&1
