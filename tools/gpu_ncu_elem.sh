cd $GRAFT_REPO_ROOT
python tools/one_apply.py --level 5 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_elem_ -s 1 -c 1 -o gpurun_out/prof_elem python tools/one_apply.py --level 5 > gpurun_out/ncu.log 2>&1
