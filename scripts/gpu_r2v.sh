cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "step or trajectory or large or edge" > gpurun_out/r2v_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2v_pytest.log
timeout 600 python scripts/late_window_launches.py 4 990 3 > gpurun_out/r2v_late_plain.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2v_late_launches.csv python scripts/late_window_launches.py 4 990 3 > gpurun_out/r2v_late.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2v_bench4.log 2> gpurun_out/r2v_bench4.err
timeout 900 python bench.py --config 5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2v_bench5.log 2> gpurun_out/r2v_bench5.err
timeout 900 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2v_bench3.log 2> gpurun_out/r2v_bench3.err
echo done >> gpurun_out/r2v_pytest.log
