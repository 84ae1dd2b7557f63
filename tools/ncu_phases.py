"""Stall samples / executed instructions of an ncu source page (--print-source sass,cuda), aggregated per
CUDA source line and then per phase (line ranges given as name=a-b): python tools/ncu_phases.py rep file.cu
name=a-b ..."""
import csv, io, subprocess, sys, collections
rep, fname = sys.argv[1], sys.argv[2]
phases = [(p.split('=')[0], *map(int, p.split('=')[1].split('-'))) for p in sys.argv[3:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
cur, hdr = None, None
per = collections.defaultdict(lambda: [0.0, 0.0])
tot = [0.0, 0.0]
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        cur = row[1]; continue
    if row[0] == "Line No":
        hdr = row; iS = hdr.index("Warp Stall Sampling (All Samples)"); iI = hdr.index("Instructions Executed"); continue
    if hdr is None or row[0] in ("", "Function Name") or row[2] != "-":
        continue
    try:
        s, i = float(row[iS]), float(row[iI])
    except ValueError:
        continue
    tot[0] += s; tot[1] += i
    if cur and cur.endswith(fname):
        per[int(row[0])][0] += s; per[int(row[0])][1] += i
print(f"total stall samples {tot[0]:.0f}, warp instructions {tot[1]:.0f} (all files)")
acc = collections.defaultdict(lambda: [0.0, 0.0])
for ln, (s, i) in per.items():
    name = next((n for n, a, b in phases if a <= ln <= b), "other-lines")
    acc[name][0] += s; acc[name][1] += i
acc["other-files"] = [tot[0] - sum(v[0] for v in per.values()), tot[1] - sum(v[1] for v in per.values())]
for n, (s, i) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    print(f"{n:24s} stall {100 * s / tot[0]:5.1f}%   inst {100 * i / tot[1]:5.1f}%")
