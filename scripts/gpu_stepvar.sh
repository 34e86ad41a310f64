# bench variants of the step's stream layout (cfg 4, cfg 5)
TAG=${1:-sv}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "step_host or runner or nccl or step_parity" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
B="python bench.py --steps 500 --warmup 10 --no-cpu-baseline"
for v in "X=1" "TSNET_FIELD_PRIORITY=1" "X=1"; do
  echo "cfg4 $v $(env $v timeout 600 $B --config 4 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],4), round(d["roofline"]["kernel_ms"],4), d["e2e"]["value"])')" >> gpurun_out/${TAG}.log
done
echo "cfg5 $(timeout 600 $B --config 5 --no-e2e 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],4), round(d["roofline"]["kernel_ms"],4))')" >> gpurun_out/${TAG}.log
