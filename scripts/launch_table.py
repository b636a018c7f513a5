"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name:
count, total and mean duration, share of the total.  Usage: launch_table.py F [skip_first_n]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg = collections.defaultdict(lambda: [0, 0.0])
n = 0
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    n += 1
    if n <= skip:
        continue
    a = agg[r[ki][:80]]
    a[0] += 1
    a[1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{n - skip} launches, {tot / 1e3:.1f} us total")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{t / tot:6.1%} {t / 1e3:9.1f} us {c:5d} x {t / c / 1e3:8.2f} us  {k}")
