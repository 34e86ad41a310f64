# one compute-sanitizer tool per call (B200_PROFILING.md): TOOL = memcheck | racecheck | synccheck
TOOL=${1:-memcheck}; TAG=${2:-san}; cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool $TOOL --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_attr_cb.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider \
  -k "(configs and 1-) or (edge_patterns and (7-tiny or 8193 or hub_and_empty or short_rows)) or unaligned or step_parity_common_state or ten_iterations or edge_cases" \
  > gpurun_out/${TAG}_${TOOL}.log 2>&1
echo "exit $?" >> gpurun_out/${TAG}_${TOOL}.log
