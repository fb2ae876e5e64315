"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
gi = hdr.index("Grid Size") if "Grid Size" in hdr else None
agg = defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", ""))
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"total kernel time {tot / 1e6:.3f} ms over {sum(c for c, _ in agg.values())} launches (ns units)")
for name, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t / tot * 100:6.2f}%  {t / 1e6:9.3f} ms  {c:6d} launches  avg {t / c / 1e3:8.2f} us  {name}")
