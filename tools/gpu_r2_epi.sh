# validate the fused smoother epilogue: its tests, smoke, A/B V-cycle time, bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_epi.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_epi.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for i in 1 2; do
timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/epi_ab.jsonl 2>&1
HHG_NO_EPI=1 timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/epi_ab.jsonl 2>&1
done
HHG_CLOCKS_RAW=gpurun_out/clocks_raw.csv timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
