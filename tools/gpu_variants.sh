# time epsilon_apply at L5/L6 for the main build and every variant in lib/variants
cd $GRAFT_REPO_ROOT
for v in "" $(ls paper_2506_04157_b200/lib/variants/*.so 2>/dev/null); do
  for L in 5 6; do HHG_LIB=$v timeout 300 python tools/time_apply.py --level $L >> gpurun_out/time_apply.log 2>&1; done
done
