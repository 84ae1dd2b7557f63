cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_coarse.py -v -s > gpurun_out/pytest_coarse.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_coarse.log
for v in "" 1; do HHG_NO_CCL=$v timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/vcycle_ab.log 2>&1; done
HHG_CCL_GLOBAL=1 timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/vcycle_ab.log 2>&1
export HHG_STATS=1
run() { echo "### $*" >> gpurun_out/stokes_L3.jsonl; timeout 300 python tools/stokes_bench.py --level 3 --max-iters 80 --restart 80 "$@" >> gpurun_out/stokes_L3.jsonl 2>&1; }
run --l-eta 2 --tol-A 1e-4
run --l-eta 2 --tol-vbfbt 1e-2
run --l-eta 2 --tol-A 1e-6 --tol-vbfbt 1e-3 --coarse-tol 1e-8 --coarse-iters 20000
run --l-eta 2 --schur mass
run --l-eta 2 --contrast 1e4 --jump 10
run --l-eta 1
run
