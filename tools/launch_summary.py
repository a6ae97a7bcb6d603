"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: share per kernel."""
import collections
import csv
import sys

path = sys.argv[1]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, mi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Name')
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
        continue
    name = r[ki].split('(')[0][:72]
    v = float(r[vi].replace(',', ''))
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"kernel time per step {tot / steps / 1e6:.3f} ms, launches/step {sum(a[0] for a in agg.values()) / steps:.0f}")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]:
    print(f"{v / tot * 100:6.2f}%  {v / steps / 1e3:9.1f} us/step  n={n / steps:5.0f}/step  {k}")
