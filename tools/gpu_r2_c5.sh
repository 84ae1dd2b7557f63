cd $GRAFT_REPO_ROOT
timeout 300 python tools/ccl_timing.py --level 3 > gpurun_out/ccl_timing.log 2>&1
export HHG_STATS=1
run() { echo "### $*" >> gpurun_out/stokes_L3.jsonl; timeout 300 python tools/stokes_bench.py --level 3 --max-iters 60 --restart 60 --l-eta 2 --tol-A 1e-4 "$@" >> gpurun_out/stokes_L3.jsonl 2>&1; }
run --omega 1.0
run --omega 0.1
run --omega 0.03
run --uzawa adjoint
run --schur wbfbt --omega 0.0125
run --schur wbfbt --omega 0.0125 --a-r 10
