TAG=${1:-fu}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -x --timeout 900 -p no:cacheprovider -k "sell or shards or step_host or step_parity or runner" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
B="python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e"
for v in "X=1" "TSNET_FUSED_MOVE=0"; do for cfg in 5 3; do echo "cfg$cfg $v $(env $v timeout 600 $B --config $cfg 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],4), round(d["roofline"]["kernel_ms"],4))')" >> gpurun_out/${TAG}.log; done; done
