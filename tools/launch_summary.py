#!/usr/bin/env python3
"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
        k = r[hdr.index("Kernel Name")].split("(")[0]
        v = float(r[hdr.index("Metric Value")].replace(",", "")) * scale[r[hdr.index("Metric Unit")]]
        agg[k][0] += 1
        agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>11s} {'avg_us':>9s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[-60:]:60s} {v[0]:8d} {v[1]:11.1f} {v[1] / v[0]:9.2f} {v[1] / tot:6.3f}")
print(f"{'total':60s} {sum(v[0] for v in agg.values()):8d} {tot:11.1f}")
