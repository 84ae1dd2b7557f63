cd $GRAFT_REPO_ROOT
python tools/one_vcycle.py --level 5 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vcycle.csv python tools/one_vcycle.py --level 5 > gpurun_out/ncu_ll.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_elem.ncu-rep > /dev/null 2>&1
python tools/one_apply.py --level 5 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_elem_ -s 1 -c 1 -o gpurun_out/prof_elem python tools/one_apply.py --level 5 > gpurun_out/ncu.log 2>&1
