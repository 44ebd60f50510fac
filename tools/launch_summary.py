"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi = h.index('Kernel Name'), h.index('Metric Value')
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) > vi:
        try:
            v = float(r[vi].replace(',', ''))
        except ValueError:
            continue
        agg[r[ki][:100]][0] += 1
        agg[r[ki][:100]][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'launches':>8} {'total us':>10} {'per launch us':>13} {'share':>6}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:8d} {v[1] / 1e3:10.1f} {v[1] / 1e3 / v[0]:13.1f} {100 * v[1] / tot:5.1f}%  {k}")
