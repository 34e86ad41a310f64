TAG=${1:-wv}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attr_cb.py tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "csr or step_host or grad_parity_full or ragged or edge" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
B="python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e"
for v in "X=1" "TSNET_SELL_WAVES=4" "TSNET_SELL_WAVES=16"; do for cfg in 5 3; do
  echo "cfg$cfg $v $(env $v timeout 600 $B --config $cfg 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],4), round(d["roofline"]["kernel_ms"],4))')" >> gpurun_out/${TAG}.log
done; done
for c in 8 4; do echo "e2e chunks=$c $(TSNET_HOST_CHUNKS=$c timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["e2e"]["value"],1))')" >> gpurun_out/${TAG}.log; done
