# bench variants of the step's stream layout (cfg 4 and 5)
TAG=${1:-sv}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e"
for cfg in 4 5; do
  for v in "X=1" "TSNET_FIELD_PRIORITY=0" "TSNET_FIELD_STREAM=0"; do
    echo "cfg$cfg $v $(env $v timeout 600 $B --config $cfg 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],4), round(d["roofline"]["kernel_ms"],4))')" >> gpurun_out/${TAG}.log
  done
done
