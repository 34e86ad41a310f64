cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tree.py tests/test_gpu_shards.py -q -x -p no:cacheprovider > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2u_pytest.log
timeout 600 python scripts/late_window_launches.py 4 990 3 > gpurun_out/r2u_late_plain.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2u_late_launches.csv python scripts/late_window_launches.py 4 990 3 > gpurun_out/r2u_late.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2u_bench4.log 2> gpurun_out/r2u_bench4.err
echo done >> gpurun_out/r2u_pytest.log
