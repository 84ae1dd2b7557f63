# round 2: does a (nearly) exact, i.e. linear, coarse solve fix the V-BFBT inner CG / FGMRES stall at 1e6 contrast?
cd $GRAFT_REPO_ROOT
export HHG_STATS=1
timeout 900 python tools/stokes_bench.py --level 4 --max-iters 10 --l-eta 2 --coarse-tol 1e-12 --coarse-iters 20000 >> gpurun_out/stokes_lin.jsonl 2>&1
timeout 900 python tools/stokes_bench.py --level 4 --max-iters 10 --l-eta 3 --l-min 2 --coarse-tol 1e-12 --coarse-iters 20000 >> gpurun_out/stokes_lin.jsonl 2>&1
