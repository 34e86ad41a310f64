#!/bin/bash
# one call: GPU tests (optionally -k EXPR), bench cfg 4 (no CPU baseline), median-window launch lists (cfg 4 and 5)
# usage: bash scripts/gpu_check.sh TAG [pytest -k expr|all|none] [bench5]
T=${1:-chk}; K=${2:-all}; B5=${3:-}
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ "$K" = all ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
elif [ "$K" != none ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$K" > gpurun_out/${T}_pytest.log 2>&1
fi
[ -f gpurun_out/${T}_pytest.log ] && tail -2 gpurun_out/${T}_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench4.log 2> gpurun_out/${T}_bench4.err
python - <<PY
import json
d=json.loads(open("gpurun_out/${T}_bench4.log").read().strip().splitlines()[-1])
print("cfg4", round(d["value"],1), "it/s", "ms/step", round(d["ms_per_step"],4), "spmv", round(d["roofline"]["kernel_ms"],4), "frac", round(d["roofline"]["frac"],4), "e2e", round(d["e2e"]["value"],1) if d.get("e2e") else None)
print([round(w["ms_per_step"],4) for w in d["run"]["windows"]])
PY
if [ -n "$B5" ]; then
  timeout 900 python bench.py --config 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench5.log 2> gpurun_out/${T}_bench5.err
  python - <<PY
import json
d=json.loads(open("gpurun_out/${T}_bench5.log").read().strip().splitlines()[-1])
print("cfg5", round(d["value"],1), "it/s", "ms/step", round(d["ms_per_step"],4), "spmv", round(d["roofline"]["kernel_ms"],4), "frac", round(d["roofline"]["frac"],4))
print([round(w["ms_per_step"],4) for w in d["run"]["windows"]])
PY
fi
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_med4.csv python scripts/late_window_launches.py 4 584 3 > gpurun_out/${T}_med4.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_med4.csv gpurun_out/${T}_med4.txt
if [ -n "$B5" ]; then
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_med5.csv python scripts/late_window_launches.py 5 584 3 > gpurun_out/${T}_med5.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/${T}_med5.csv gpurun_out/${T}_med5.txt
fi
