# A/B timing on one B200 (the round-2 experiments in DESIGN.md §6 were run this way):
#   bash tools/build_variant.sh NAME "-DFLAG ..."     (here, before the gpurun call)
#   gpurun -- 'bash tools/gpu_ab.sh NAME [LEVEL]'    element kernel + V-cycle, product library vs exp_NAME.so
# Env switches need no variant build: HHG_NO_SPLIT=1, HHG_EPI=1, HHG_NO_FX=1, HHG_NO_CCL=1 (time_vcycle.py / time_elem.py).
cd $GRAFT_REPO_ROOT
NAME=$1; L=${2:-5}
for i in 1 2; do
  timeout 300 python tools/time_elem.py --level $L >> gpurun_out/ab_elem.jsonl 2>&1
  HHG_LIB=$GRAFT_REPO_ROOT/paper_2506_04157_b200/lib/exp_$NAME.so timeout 300 python tools/time_elem.py --level $L >> gpurun_out/ab_elem.jsonl 2>&1
done
timeout 300 python tools/time_vcycle.py --level $L >> gpurun_out/ab_vc.jsonl 2>&1
HHG_LIB=$GRAFT_REPO_ROOT/paper_2506_04157_b200/lib/exp_$NAME.so timeout 300 python tools/time_vcycle.py --level $L >> gpurun_out/ab_vc.jsonl 2>&1
