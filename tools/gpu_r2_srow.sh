# shared row-start table in k_elem_fp: quick element parity + A/B element-kernel timing vs the HHG_EXP_NOSROW build
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config1 or stokes_apply or diag_and_dot or sampled_rows or edge_cases or quadrature_point_viscosity_apply or vcycle_matches_oracle" > gpurun_out/pytest_srow.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_srow.log
for i in 1 2; do for L in 4 5; do
  timeout 300 python tools/time_elem.py --level $L >> gpurun_out/srow_elem.jsonl 2>&1
  HHG_LIB=$GRAFT_REPO_ROOT/paper_2506_04157_b200/lib/exp_nosrow.so timeout 300 python tools/time_elem.py --level $L >> gpurun_out/srow_elem.jsonl 2>&1
done; done
timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/srow_vc.jsonl 2>&1
