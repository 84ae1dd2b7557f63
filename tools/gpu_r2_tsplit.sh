# k_elem_fp with kWT = 2 type groups (4 warps per brick): element parity subset + A/B element-kernel timing
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config1 or stokes_apply or diag_and_dot or sampled_rows or edge_cases or quadrature_point_viscosity_apply or vcycle_matches_oracle or mass_apply or buoyancy" > gpurun_out/pytest_tsplit.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tsplit.log
for i in 1 2; do for L in 4 5; do
  timeout 300 python tools/time_elem.py --level $L >> gpurun_out/tsplit_elem.jsonl 2>&1
  HHG_LIB=$GRAFT_REPO_ROOT/paper_2506_04157_b200/lib/exp_tsplit1.so timeout 300 python tools/time_elem.py --level $L >> gpurun_out/tsplit_elem.jsonl 2>&1
done; done
timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/tsplit_vc.jsonl 2>&1
HHG_LIB=$GRAFT_REPO_ROOT/paper_2506_04157_b200/lib/exp_tsplit1.so timeout 300 python tools/time_vcycle.py --level 5 >> gpurun_out/tsplit_vc.jsonl 2>&1
