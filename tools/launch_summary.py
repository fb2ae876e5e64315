"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in data:
    k = d["Kernel Name"][:70]
    m, v = d["Metric Name"], float(d["Metric Value"].replace(",", ""))
    if m == "gpu__time_duration.sum":
        agg[k][0] += 1
        agg[k][1] += v
    elif "dram__bytes" in m:
        agg[k][2] += v
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    gbs = a[2] / a[1] if a[1] else 0.0
    print(f"{k:70s} n={a[0]:6d} t={a[1] / 1e3:10.1f}us ({100 * a[1] / tot:5.1f}%) avg={a[1] / a[0] / 1e3:8.2f}us GB/s={gbs:8.1f}")
print(f"total {tot / 1e3:.1f} us over {sum(a[0] for a in agg.values())} launches")
