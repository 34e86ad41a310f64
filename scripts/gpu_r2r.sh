# full GPU test suite + bench (cfg 4) with the new plan choice
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 1200 > gpurun_out/r2r_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2r_pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2r_bench4.log 2> gpurun_out/r2r_bench4.err; echo "rc=$?" >> gpurun_out/r2r_bench4.err
