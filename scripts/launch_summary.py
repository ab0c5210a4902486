"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if len(r) <= vi or not r[vi]:
        continue
    us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0][:80]
    agg[name][0] += 1
    agg[name][1] += us
tot = sum(v for _, v in agg.values())
print(f"total GPU time {tot / 1e3:.2f} ms over {sum(c for c, _ in agg.values())} launches")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{v / 1e3:9.3f} ms {100 * v / tot:5.1f}%  n={c:5d}  avg {v / c:9.1f} us  {k}")
