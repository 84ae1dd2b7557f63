"""Summarise an ncu launch-list CSV (gpu__time_duration.sum) after the last separator kernel."""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; iN = h.index('Kernel Name'); iV = h.index('Metric Value'); iID = h.index('ID')
ks = [(int(r[iID]), r[iN], float(r[iV].replace(',', ''))) for r in rows[hi + 1:] if len(r) > iV]
sep = [j for j, k in enumerate(ks) if 'at::' in k[1] and 'Mul' in k[1]]
if sep and '--after-sep' in sys.argv:
    ks = [k for k in ks[sep[-1] + 1:] if 'at::' not in k[1]]
def short(n):
    n = re.sub(r'\(.*', '', n); n = re.sub(r'^void ', '', n)
    return n.replace('hhg::', '')[:60]
tot = collections.Counter(); cnt = collections.Counter()
for _, n, v in ks:
    tot[short(n)] += v; cnt[short(n)] += 1
T = sum(tot.values())
print(f"kernels={len(ks)} total={T/1e6:.3f} ms")
for k, v in tot.most_common(25):
    print('%-62s %8.3f ms %5.1f%%  n=%d' % (k, v / 1e6, 100 * v / T, cnt[k]))
