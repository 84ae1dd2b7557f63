cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_partition.py -m gpu -q > gpurun_out/pytest_edge.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_edge.log
timeout 1500 python tools/stokes_bench.py --level 5 --l-eta 2 --max-iters 40 --restart 40 > gpurun_out/stokes_L5.jsonl 2>&1
