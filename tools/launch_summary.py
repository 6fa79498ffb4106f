"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel launches, time, share."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':45s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:45]:45s} {n:8d} {t / 1e6:10.3f} {t / tot * 100:6.1f}%")
print(f"{'TOTAL':45s} {sum(v[0] for v in agg.values()):8d} {tot / 1e6:10.3f}")
