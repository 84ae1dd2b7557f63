# round 2: cluster coarse PCG (compile-time cluster dims) + batched inner-CG checks
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_coarse.py -v -s > gpurun_out/pytest_coarse.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_coarse.log
for v in "" 1; do HHG_NO_CCL=$v timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/vcycle_ab.log 2>&1; done
timeout 300 python tools/one_vcycle.py --level 5 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vcycle.csv python tools/one_vcycle.py --level 5 > gpurun_out/ncu_ll.log 2>&1
HHG_STATS=1 timeout 600 python tools/stokes_bench.py --level 4 --max-iters 40 --l-eta 2 >> gpurun_out/stokes_diag.jsonl 2>&1
