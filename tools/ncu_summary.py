"""Key counters of every kernel in an ncu report: python tools/ncu_summary.py <rep>"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.per_cycle_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'smsp__inst_executed.sum',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct',
        'sm__cycles_elapsed.avg.per_second', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'smsp__sass_thread_inst_executed_op_dfma_pred_on.sum', 'smsp__sass_thread_inst_executed_op_dadd_pred_on.sum',
        'smsp__sass_thread_inst_executed_op_dmul_pred_on.sum',
        'smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed', 'smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed',
        'smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed', 'smsp__cycles_elapsed.avg',
        'launch__block_size', 'launch__grid_size']
for v in rows[2:]:
    print('==', v[h.index('Kernel Name')][:90], 'grid', v[h.index('launch__grid_size')] if 'launch__grid_size' in h else '')
    for w in want:
        if w in h:
            i = h.index(w); print(f"{w:70s} {u[i]:8s} {v[i]}")
    st = sorted(((float(v[i]), h[i]) for i in range(len(h)) if h[i].startswith('smsp__average_warps_issue_stalled')
                 and h[i].endswith('per_issue_active.ratio')), reverse=True)
    for val, name in st[:12]:
        print(f"{name.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):40s} {val:.3f}")
