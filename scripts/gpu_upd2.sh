TAG=${1:-u2}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 env TSNET_UPDATE=2,1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "step or ten_iter or runner or shards or trajectory" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
B="python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e"
for v in "TSNET_UPDATE=2,0" "TSNET_UPDATE=2,1" "TSNET_UPDATE=1,1" "TSNET_UPDATE=1,0"; do for cfg in 5 4; do
  echo "cfg$cfg $v $(env $v timeout 600 $B --config $cfg 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],4))')" >> gpurun_out/${TAG}.log
done; done
