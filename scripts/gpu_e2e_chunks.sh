TAG=${1:-e2ec}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in 8 10 12 16 8 12; do echo "bench chunks=$c $(TSNET_HOST_CHUNKS=$c timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["e2e"]["value"],1))')" >> gpurun_out/${TAG}.log; done
