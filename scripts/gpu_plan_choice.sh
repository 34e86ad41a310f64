TAG=${1:-pc}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e"
for a in "--config 3 --plan csr" "--config 3 --plan sell" "--config 5 --plan sell" "--config 2 --plan csr" "--config 2 --plan sell"; do
  echo "$a $(timeout 600 $B $a 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],4), round(d["roofline"]["kernel_ms"],4))')" >> gpurun_out/${TAG}.log
done
for a in "--config 3 --plan sell" ; do echo "MINB3 $a $(TSNET_SELL=g4,4,3 timeout 600 $B $a 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],4), round(d["roofline"]["kernel_ms"],4))')" >> gpurun_out/${TAG}.log; done
