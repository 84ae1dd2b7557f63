"""Per-(kernel, grid) breakdown of an ncu launch list between the last two torch separator kernels:
python tools/launch_levels.py <launches.csv> [top]"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; iN = h.index('Kernel Name'); iV = h.index('Metric Value'); iG = h.index('Grid Size')
ks = [(r[iN], float(r[iV].replace(',', '')), r[iG]) for r in rows[hi + 1:] if len(r) > iV]
sep = [j for j, k in enumerate(ks) if 'at::' in k[0]]
if len(sep) >= 2:
    ks = ks[sep[-2] + 1:sep[-1]]
ks = [k for k in ks if 'at::' not in k[0]]
d = collections.defaultdict(list)
for n, v, g in ks:
    n = re.sub(r'\(.*', '', n).replace('void ', '').replace('hhg::', '')[:30]
    d[(n, g)].append(v)
tot = sum(v for _, v, _ in ks)
print(f"kernels={len(ks)} total={tot/1e6:.3f} ms")
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1]))[:top]:
    print(f"{k[0]:30s} {k[1]:16s} n={len(v):4d} avg={sum(v)/len(v)/1e3:8.1f}us tot={sum(v)/1e6:.3f}ms {100*sum(v)/tot:5.1f}%")
