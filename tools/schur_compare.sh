# Schur-approximation / Uzawa comparison (P:664-685 qualitatively) on one B200: shell(3,2) L4,
# contrast 1e4 x 10, buoyancy rhs, FGMRES to 1e-8 relative or 40 iterations.
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_wbfbt.py -m gpu -q -k "fgmres or rejects" > gpurun_out/pytest_wbfbt2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_wbfbt2.log
O=gpurun_out/schur_compare.jsonl
B="timeout 600 python tools/stokes_bench.py --level 4 --contrast 1e4 --jump 10 --max-iters 40 --restart 40"
$B --schur vbfbt >> $O 2>&1
$B --schur mass >> $O 2>&1
$B --schur wbfbt --omega 0.0125 >> $O 2>&1
$B --schur wbfbt --omega 0.3 >> $O 2>&1
$B --schur wbfbt --omega 0.0125 --a-r 10 --a-l 1 >> $O 2>&1
$B --schur vbfbt --uzawa inexact --tol-A 1e-4 >> $O 2>&1
$B --schur vbfbt --uzawa adjoint --tol-A 1e-4 >> $O 2>&1
