"""Per-colour table of a relaxation sweep from an ncu launch list
(gpu__time_duration.sum + dram bytes): the relax_task_kernel<*, true> launches
of ONE sweep in order, bucketed by duration.

    python tools/relax_colour_table.py launches.csv
"""
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
by_id = {}
for d in data:
    e = by_id.setdefault(d["ID"], {"name": d["Kernel Name"], "grid": d.get("Grid Size", ""), "t": 0.0, "bytes": 0.0})
    v = float(d["Metric Value"].replace(",", ""))
    if d["Metric Name"] == "gpu__time_duration.sum":
        e["t"] = v / 1e3
    elif "dram__bytes" in d["Metric Name"]:
        e["bytes"] += v
launches = [by_id[k] for k in sorted(by_id, key=int)]
sweep = [e for e in launches if "relax_task_kernel" in e["name"] and ("true" in e["name"] or ", 1>" in e["name"])]
print(f"{len(launches)} launches, {len(sweep)} coloured-sweep launches, total {sum(e['t'] for e in launches) / 1e3:.2f} ms")
buckets = [(0, 5), (5, 10), (10, 20), (20, 50), (50, 100), (100, 1000), (1000, 1e9)]
for lo, hi in buckets:
    sel = [e for e in sweep if lo <= e["t"] < hi]
    if sel:
        print(f"  {lo:>5}-{hi:<6g} us: {len(sel):6d} launches, {sum(e['t'] for e in sel) / 1e3:9.2f} ms, "
              f"{sum(e['bytes'] for e in sel) / 1e9:8.2f} GB")
print("first 40 sweep launches (us, grid, MB):")
for e in sweep[:40]:
    print(f"  {e['t']:9.2f} {e['grid']:>16} {e['bytes'] / 1e6:10.2f}")
other = {}
for e in launches:
    if e in sweep:
        continue
    k = e["name"][:60]
    o = other.setdefault(k, [0, 0.0])
    o[0] += 1
    o[1] += e["t"]
for k, (n, t) in sorted(other.items(), key=lambda x: -x[1][1])[:12]:
    print(f"  {k:60s} n={n:6d} t={t / 1e3:9.2f} ms")
