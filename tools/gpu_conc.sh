# A/B of the concurrent sparse-brick launch (side stream; HHG_NO_CONC=1 = serial launches) + a parity subset
cd $GRAFT_REPO_ROOT
for i in 1 2; do
  timeout 300 python tools/time_elem.py --level 5 >> gpurun_out/conc_elem.jsonl 2>&1
  HHG_NO_CONC=1 timeout 300 python tools/time_elem.py --level 5 >> gpurun_out/conc_elem.jsonl 2>&1
done
for L in 4 3; do
  timeout 300 python tools/time_elem.py --level $L >> gpurun_out/conc_elem.jsonl 2>&1
  HHG_NO_CONC=1 timeout 300 python tools/time_elem.py --level $L >> gpurun_out/conc_elem.jsonl 2>&1
done
timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/conc_vc.jsonl 2>&1
HHG_NO_CONC=1 timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/conc_vc.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_robustness.py tests/test_gpu_multirank.py -m gpu -q -x -k "config1 or shell_level2 or vcycle_matches_oracle or host_batch or robust or hierarch or config3_full or multirank or rank or divT" > gpurun_out/conc_parity.log 2>&1; echo "rc=$?" >> gpurun_out/conc_parity.log
