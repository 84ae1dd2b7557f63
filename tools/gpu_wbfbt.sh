cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_wbfbt.py -m gpu -q -x > gpurun_out/pytest_wbfbt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_wbfbt.log
