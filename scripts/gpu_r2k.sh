cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in base nopf lanepf ldca ldnc lanepf_ldca diag1 diag2; do
  timeout 300 python scripts/tile_variant_probe.py 4 $v >> gpurun_out/r2k_variants.log 2>&1
done
echo done >> gpurun_out/r2k_variants.log
