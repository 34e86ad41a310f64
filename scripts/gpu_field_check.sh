TAG=${1:-fc}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shards.py -m gpu -q -x --timeout 900 -p no:cacheprovider -k "not config4_full and not config5_full and not build_P" > gpurun_out/${TAG}_pytest.log 2>&1; echo "exit $?" >> gpurun_out/${TAG}_pytest.log
B="python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-e2e"
for cfg in 4 5 3; do echo "cfg$cfg $(timeout 600 $B --config $cfg 2>/dev/null | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],4), round(d["roofline"]["kernel_ms"],4))')" >> gpurun_out/${TAG}.log; done
B5="python bench.py --config 5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -s 3000 -c 200 --csv --log-file gpurun_out/${TAG}_warm5.csv $B5 > gpurun_out/${TAG}_ncu5.log 2>&1
