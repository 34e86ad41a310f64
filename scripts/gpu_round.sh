# round-1 call 2: tests, SpMV probe, bench on cfg 4 + cfg 5, ncu of k_spmv
set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -k "trajectory or step_parity or runner or edge or ragged or config4_sampled" > gpurun_out/r2_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2_pytest_gpu.log
timeout 600 python scripts/spmv_probe.py 4 > gpurun_out/r2_probe4.log 2>&1
timeout 900 python scripts/spmv_probe.py 5 > gpurun_out/r2_probe5.log 2>&1
timeout 900 python bench.py --steps 300 --warmup 10 --pre-iters 500 --no-cpu-baseline > gpurun_out/r2_bench4.log 2>&1
timeout 1200 python bench.py --config 5 --steps 100 --warmup 5 --pre-iters 300 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench5.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --pre-iters 10 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 5 -c 1 -o gpurun_out/r2_spmv python bench.py --steps 20 --warmup 3 --pre-iters 10 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 60 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 20 --warmup 3 --pre-iters 10 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_launch.log 2>&1
echo done
