# one gpurun call: GPU tests, bench (cfg 4), launch list + ncu full of the top kernel
# usage: bash scripts/gpu_run.sh TAG [pytest -k expr] [ncu kernel regex]
TAG=${1:-r1}
KEXPR=${2:-}
KREGEX=${3:-k_spmv2}
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${TAG}_smi.txt 2>&1
if [ -n "$KEXPR" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider -k "$KEXPR" > gpurun_out/${TAG}_pytest_gpu.log 2>&1
else
  timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1
fi
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench4.log 2>&1
echo "bench exit $?" >> gpurun_out/${TAG}_bench4.log
timeout 900 python bench.py --plan --no-cpu-baseline --no-e2e --steps 200 > gpurun_out/${TAG}_bench4_plan.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 bench.py --sharded --no-cpu-baseline --steps 200 > gpurun_out/${TAG}_bench4_sharded1.log 2>&1
timeout 1200 python bench.py --config 5 --no-cpu-baseline --no-e2e --steps 200 > gpurun_out/${TAG}_bench5.log 2>&1
B="python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s 5 -c 1 -o gpurun_out/${TAG}_top $B > gpurun_out/${TAG}_ncu.log 2>&1
echo done
B5="python bench.py --config 5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attr_sell_g -s 5 -c 1 -o gpurun_out/${TAG}_sell5 $B5 > gpurun_out/${TAG}_ncu_sell5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 400 --csv --log-file gpurun_out/${TAG}_launches5.csv $B5 > gpurun_out/${TAG}_ncu_launch5.log 2>&1
echo done5
