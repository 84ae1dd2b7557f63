# round 2: Stokes solves for the record (HHG_STATS=1 residual histories), and the L2 run compared with the oracle
cd $GRAFT_REPO_ROOT
export HHG_STATS=1
run() { echo "### $*" >> gpurun_out/stokes_final.jsonl; timeout $1 python tools/stokes_bench.py "${@:2}" >> gpurun_out/stokes_final.jsonl 2>&1; }
run 300 --level 2 --max-iters 60 --restart 60
run 600 --level 4 --contrast 1e4 --jump 10 --l-eta 2 --max-iters 60 --restart 60
run 900 --level 5 --contrast 1e4 --jump 10 --l-eta 3 --max-iters 60 --restart 60
run 900 --level 4 --l-eta 3 --tol-A 1e-4 --max-iters 80 --restart 80
run 1200 --level 5 --l-eta 4 --tol-A 1e-4 --max-iters 60 --restart 60
