# usage: bash tools/gpu_run.sh [ncu|ll]  -- GPU parity tests, apply timing at L5/L6, bench (no CPU baseline)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in "" $(ls paper_2506_04157_b200/lib/variants/*.so 2>/dev/null); do
  for L in 5 6; do HHG_LIB=$v timeout 300 python tools/time_apply.py --level $L >> gpurun_out/time_apply.log 2>&1; done
done
HHG_CLOCKS_RAW=gpurun_out/clocks_raw.csv timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ "$1" = "ncu" ]; then
  python tools/one_apply.py --level 5 > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_elem_ -s 1 -c 1 -o gpurun_out/prof_elem python tools/one_apply.py --level 5 > gpurun_out/ncu.log 2>&1
fi
if [ "$1" = "ll" ]; then
  python tools/one_vcycle.py --level 5 > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vcycle.csv python tools/one_vcycle.py --level 5 > gpurun_out/ncu_ll.log 2>&1
fi
