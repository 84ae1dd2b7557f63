# round-2 final validation on one B200: smoke, bench (+ reference arm), V-cycle launch list, ncu --set full of the
# fine-level element kernels (dense + sparse) and of the config-2 stokes_apply kernels, then all -m gpu tests
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
HHG_CLOCKS_RAW=gpurun_out/clocks_raw.csv timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
python tools/one_vcycle.py --level 5 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vcycle.csv python tools/one_vcycle.py --level 5 > gpurun_out/ncu_ll.log 2>&1
python tools/one_apply.py --level 5 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_elem_ -s 2 -c 2 -o gpurun_out/prof_elemA_L5 python tools/one_apply.py --level 5 > gpurun_out/ncu_elem.log 2>&1
python tools/one_stokes.py --level 4 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:k_elem_ -s 4 -c 2 -o gpurun_out/prof_stokes_L4 python tools/one_stokes.py --level 4 > gpurun_out/ncu_stokes.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
echo done > gpurun_out/final_done
