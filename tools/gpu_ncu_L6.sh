cd $GRAFT_REPO_ROOT
python tools/one_apply_dev.py --level 6 > gpurun_out/plain6.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_elem_fp -s 1 -c 1 -o gpurun_out/prof_elem_L6 python tools/one_apply_dev.py --level 6 > gpurun_out/ncu6.log 2>&1
echo rc=$? >> gpurun_out/ncu6.log
