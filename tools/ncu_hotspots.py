"""Per-CUDA-line hotspots from an ncu report (source page with --print-source sass,cuda) and the
SASS opcode mix: python tools/ncu_hotspots.py <rep.ncu-rep> [top]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
hi = [i for i, l in enumerate(lines) if l.startswith('"Line No"')][0]
rows = list(csv.reader(io.StringIO("\n".join(lines[hi:]))))
h = rows[0]
iS = h.index("Warp Stall Sampling (All Samples)"); iI = h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
src_rows = [r for r in rows[1:] if len(r) > iI and r[2] == "-"]      # cuda-line aggregate rows
sass_rows = [r for r in rows[1:] if len(r) > iI and r[2] != "-"]
tot_s = sum(float(r[iS] or 0) for r in src_rows); tot_i = sum(float(r[iI] or 0) for r in src_rows)
print(f"total samples {tot_s:.0f}, warp inst {tot_i:.0f}")
for r in sorted(src_rows, key=lambda r: -float(r[iS] or 0))[:top]:
    st = sorted(((float(r[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
    print(f"{100*float(r[iS] or 0)/tot_s:5.1f}% stall {100*float(r[iI] or 0)/max(tot_i,1):5.1f}% inst L{r[0]:<4} "
          f"{r[1].strip()[:70]:70s} " + " ".join(f"{n}:{v:.0f}" for v, n in st))
ops = collections.Counter(); opst = collections.Counter()
for r in sass_rows:
    op = r[3].split()[0] if r[3].split() else "?"
    if op.startswith("@"): op = r[3].split()[1]
    op = op.split(".")[0]
    ops[op] += float(r[iI] or 0); opst[op] += float(r[iS] or 0)
T = sum(ops.values())
print("opcode mix (inst %, stall %):", ", ".join(f"{k} {100*v/T:.1f}/{100*opst[k]/tot_s:.1f}" for k, v in ops.most_common(22)))
