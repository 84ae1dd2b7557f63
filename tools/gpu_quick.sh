# quick A/B: GPU parity subset + apply timing (main build and lib/variants/*.so)
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config1 or level2 or transfers_larger" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in "" $(ls paper_2506_04157_b200/lib/variants/*.so 2>/dev/null); do
  for L in 5 6; do HHG_LIB=$v timeout 300 python tools/time_apply.py --level $L >> gpurun_out/time_apply.log 2>&1; done
done
