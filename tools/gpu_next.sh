# NEXT-row checks: Stokes (all Schur variants) + w-BFBT + temperature parity, solve timings
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_temperature.py tests/test_gpu_wbfbt.py tests/test_gpu_parity.py -m gpu -q -k "temperature or stokes or wbfbt or kmg or kp1 or vmass or p1_transfers" > gpurun_out/pytest_next.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_next.log
for L in 4 5; do timeout 600 python tools/temp_bench.py --level $L >> gpurun_out/temp_bench.jsonl 2>&1; done
B="timeout 600 python tools/stokes_bench.py --level 4 --contrast 1e4 --jump 10 --max-iters 40 --restart 40"
$B --schur vbfbt >> gpurun_out/stokes_sync.jsonl 2>&1
$B --schur mass >> gpurun_out/stokes_sync.jsonl 2>&1
