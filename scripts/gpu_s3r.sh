#!/bin/bash
# session-3 call r: the step parity tests after the gains-decision change; spread tests (stray overflow)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s3r
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 900 -p no:cacheprovider -k "step or spread or teacher" > gpurun_out/${T}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
echo done
