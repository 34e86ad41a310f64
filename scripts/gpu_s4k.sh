#!/bin/bash
# session-4 call k: the field chain with programmatic dependent launches (probe build FIELD_PDL=1)
# against the product: step times at the median windows of cfg 4 / cfg 5 (graph replays), then the
# GPU suite and the bench lines with the probe build standing in for libtsnet.so on the box's scratch copy
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=s4k
V=paper_2509_19785_b200/build/variants/libtsnet_pdl.so
for rep in 1 2 3; do
  for name in product pdl; do
    timeout 300 python scripts/step_variant_probe.py 4 584 $name 200 graph 2>&1 | grep '^{' >> gpurun_out/${T}_steps.jsonl
  done
done
for rep in 1 2; do
  for name in product pdl; do
    timeout 400 python scripts/step_variant_probe.py 5 600 $name 200 graph 2>&1 | grep '^{' >> gpurun_out/${T}_steps.jsonl
  done
done
timeout 300 python scripts/step_variant_probe.py 4 584 pdl 50 eager 2>&1 | tail -3 >> gpurun_out/${T}_steps.jsonl
cp $V paper_2509_19785_b200/libtsnet.so
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${T}_pytest_gpu_pdl.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest_gpu_pdl.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke_pdl.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench4_pdl.log 2>&1
timeout 1200 python bench.py --config 5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench5_pdl.log 2>&1
echo done
