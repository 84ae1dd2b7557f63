cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition.py -m gpu -q -k "vcycle or ablock or stokes or edge or partition or rank" > gpurun_out/pytest_pcg.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pcg.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
HHG_CLOCKS_RAW=gpurun_out/clocks_raw.csv timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
python tools/one_vcycle.py --level 5 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vcycle.csv python tools/one_vcycle.py --level 5 > gpurun_out/ncu_ll.log 2>&1
