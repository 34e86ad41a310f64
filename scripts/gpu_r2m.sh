cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in base diag1; do
  timeout 300 python scripts/tile_variant_probe.py 4 $v >> gpurun_out/r2m_variants.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_attr_cb.py -q -x -p no:cacheprovider > gpurun_out/r2m_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2m_pytest.log
timeout 300 python scripts/attr_tile_probe.py 4 5 > gpurun_out/r2m_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attr_tile -s 2 -c 1 -o gpurun_out/r2m_tile python scripts/attr_tile_probe.py 4 5 > gpurun_out/r2m_ncu.log 2>&1
echo done >> gpurun_out/r2m_variants.log
