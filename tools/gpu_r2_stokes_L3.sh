# round 2: config-4 Stokes convergence study at L3 (cheap): inner tolerances, l_eta, coarse solves
cd $GRAFT_REPO_ROOT
export HHG_STATS=1
run() { echo "### $*" >> gpurun_out/stokes_L3.jsonl; timeout 420 python tools/stokes_bench.py --level 3 --max-iters 80 --restart 80 "$@" >> gpurun_out/stokes_L3.jsonl 2>&1; }
run --l-eta 2
run --l-eta 3
run --l-eta 3 --coarse-tol 1e-2 --coarse-iters 3000
run --l-eta 3 --tol-vbfbt 1e-2
run --l-eta 3 --tol-A 1e-4
run --l-eta 3 --tol-vbfbt 1e-3 --tol-A 1e-4
run --l-eta 3 --schur wbfbt --omega 0.0125
run --l-eta 3 --contrast 1e4 --jump 10
timeout 600 python tools/vcycle_spread.py --levels 3,5 > gpurun_out/vcycle_spread.jsonl 2>&1
