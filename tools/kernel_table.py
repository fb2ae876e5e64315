"""Per-kernel HBM table from an ncu --csv launch list with gpu__time_duration.sum,
dram__bytes_read.sum and dram__bytes_write.sum: launches, total time, DRAM bytes,
achieved GB/s (bytes / time) and the fraction of the measured HBM peak, for the
kernels that move at least MIN_MB per launch on average (small launches are
latency-bound by construction and are listed separately)."""
import collections
import csv
import json
import os
import sys

path = sys.argv[1]
min_mb = float(sys.argv[2]) if len(sys.argv) > 2 else 16.0
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6553.6) \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) \
    else 6553.6
rows = list(csv.reader(open(path)))
hdr, per = None, collections.defaultdict(dict)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        per[(d["ID"], d["Kernel Name"])][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])  # launches, ns, bytes, max GB/s
for (lid, name), m in per.items():
    k = name.split("(")[0].replace("void ", "").replace("lamgb::", "").replace("<unnamed>::", "")[:48]
    t = m.get("gpu__time_duration.sum", 0.0)
    by = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    a = agg[k]
    a[0] += 1
    a[1] += t
    a[2] += by
    if t > 0:
        a[3] = max(a[3], by / t)
print(f"peak {peak} GB/s (MEASURED_PEAKS.json hbm_gbs); ncu launch list {os.path.basename(path)}")
print(f"{'kernel':48s} {'launches':>8s} {'total ms':>9s} {'MB/launch':>10s} {'GB/s':>8s} {'%peak':>6s} {'best GB/s':>9s}")
big, small = [], []
for k, (n, t, by, best) in sorted(agg.items(), key=lambda x: -x[1][1]):
    line = (f"{k:48s} {n:8d} {t / 1e6:9.3f} {by / n / 1e6:10.2f} {by / t if t else 0:8.1f} "
            f"{100 * by / t / peak if t else 0:6.1f} {best:9.1f}")
    (big if by / n / 1e6 >= min_mb else small).append(line)
print("\n".join(big))
print(f"--- launches moving < {min_mb} MB on average (latency-bound) ---")
print("\n".join(small[:25]))
