# round 2: cluster coarse PCG validation + V-cycle A/B + config-4 Stokes diagnosis (HHG_STATS=1)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_coarse.py -v -s > gpurun_out/pytest_coarse.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_coarse.log
for v in "" 1; do HHG_NO_CCL=$v timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/vcycle_ab.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_robustness.py -q -x -k "vcycle or multirank or partitioned or deterministic or two_solver" > gpurun_out/pytest_vc.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_vc.log
export HHG_STATS=1
for args in "--l-eta 2" "--l-eta 2 --coarse-tol 1e-2 --coarse-iters 3000" "--l-eta 3 --l-min 2 --coarse-tol 1e-2 --coarse-iters 3000"; do
  timeout 400 python tools/stokes_bench.py --level 4 --max-iters 40 $args >> gpurun_out/stokes_diag.jsonl 2>&1
done
