"""Per-launch counters of the element kernel from an ncu report -> JSON (read by bench.py for the
roofline): duration, DRAM bytes, thread-level DFMA / DADD / DMUL counts and flops per micro tet
(DFMA = 2 flops); several captured kernels (one operator application split over launches) are summed.
python tools/ncu_counts.py <rep.ncu-rep> <n_tets> <label> > profiles/<out>.json"""
import csv, io, json, subprocess, sys
rep, n_tets, label = sys.argv[1], int(sys.argv[2]), sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
res = []
for v in rows[2:]:
    d = dict(zip(h, v))
    num = lambda k: float(d[k].replace(",", "")) if d.get(k) not in (None, "", "n/a") else None
    def unit_scale(k):
        un = u[h.index(k)] if k in h else ""
        return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3,
                "nsecond": 1e-9, "second": 1, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}.get(un, 1)
    def count(op):
        # thread-instruction count: the .sum metric when it was collected, else (--set full alone) the
        # .sum.per_cycle_elapsed rate times the elapsed SMSP cycles it is normalised by
        c = num("smsp__sass_thread_inst_executed_op_%s_pred_on.sum" % op)
        if c is None:
            r = num("smsp__sass_thread_inst_executed_op_%s_pred_on.sum.per_cycle_elapsed" % op)
            cyc = num("smsp__cycles_elapsed.avg")
            c = round(r * cyc) if r is not None and cyc is not None else None
        return c
    dfma, dadd, dmul = count("dfma"), count("dadd"), count("dmul")
    dur = num("gpu__time_duration.sum") * unit_scale("gpu__time_duration.sum")
    rd = num("dram__bytes_read.sum") * unit_scale("dram__bytes_read.sum")
    wr = num("dram__bytes_write.sum") * unit_scale("dram__bytes_write.sum")
    res.append({"label": label, "kernel": d.get("Kernel Name", "")[:160], "n_tets": n_tets, "duration_s": dur,
                "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes": rd + wr,
                "dfma": dfma, "dadd": dadd, "dmul": dmul,
                "flops_per_tet": (2 * dfma + dadd + dmul) / n_tets if dfma is not None else None,
                "fp64_pipe_active_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                "warps_active_per_sm": num("sm__warps_active.avg.per_cycle_active"),
                "registers": num("launch__registers_per_thread"), "source": rep})
if len(res) == 1:
    print(json.dumps(res[0], indent=1))
else:
    # several kernels captured for one operator application (e.g. k_elem_fp over the dense bricks + k_elem_sparse
    # over the sparse ones): the operator's counters are their sums, duration the sum of the launch durations
    tot = {"label": label, "kernel": " + ".join(r["kernel"].split("(")[0] for r in res), "n_tets": n_tets}
    for k in ("duration_s", "dram_read_bytes", "dram_write_bytes", "dram_bytes", "dfma", "dadd", "dmul"):
        tot[k] = sum(r[k] for r in res)
    tot["flops_per_tet"] = (2 * tot["dfma"] + tot["dadd"] + tot["dmul"]) / n_tets
    tot["source"] = rep
    tot["parts"] = res
    print(json.dumps(tot, indent=1))
