cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in base pref1 pref6 pref3c16 pref6c4 l2b256 pref6l2 base; do
  timeout 300 python scripts/tile_variant_probe.py 4 $v >> gpurun_out/r2t_variants.log 2>&1
done
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2t_late_launches.csv python scripts/late_window_launches.py 4 990 3 > gpurun_out/r2t_late.log 2>&1
echo done >> gpurun_out/r2t_variants.log
