# full GPU check: all -m gpu tests, smoke, bench (with cpu_baseline), launch list, ncu of the element kernel
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python tools/max_size.py > gpurun_out/max_size.log 2>&1; echo "max_size rc=$?" >> gpurun_out/max_size.log
for L in 4 5; do timeout 600 python tools/temp_bench.py --level $L >> gpurun_out/temp_bench.jsonl 2>&1; done
HHG_CLOCKS_RAW=gpurun_out/clocks_raw.csv timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
python tools/one_vcycle.py --level 5 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vcycle.csv python tools/one_vcycle.py --level 5 > gpurun_out/ncu_ll.log 2>&1
python tools/one_apply.py --level 5 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_elem_ -s 1 -c 1 -o gpurun_out/prof_elem python tools/one_apply.py --level 5 > gpurun_out/ncu.log 2>&1
