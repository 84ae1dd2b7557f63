# sparse-brick kernel split: element parity tests, element-kernel and V-cycle A/B (HHG_NO_SPLIT=1 = old path)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py -m gpu -q -x > gpurun_out/pytest_split.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_split.log
for L in 3 4 5; do
  timeout 300 python tools/time_elem.py --level $L >> gpurun_out/split_elem.jsonl 2>&1
  HHG_NO_SPLIT=1 timeout 300 python tools/time_elem.py --level $L >> gpurun_out/split_elem.jsonl 2>&1
done
for i in 1 2; do
timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/split_vc.jsonl 2>&1
HHG_NO_SPLIT=1 timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/split_vc.jsonl 2>&1
done
