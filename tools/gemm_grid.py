"""GEMM launches of an ncu launch list (gpu__time_duration.sum, launch__grid_size)
grouped by kernel and grid: total / count / mean.  Usage: gemm_grid.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
recs = {}
for r in rows:
    if len(r) != len(hdr) or r[0] == "ID":
        continue
    d = dict(zip(hdr, r))
    v = recs.setdefault(d["ID"], {"name": d["Kernel Name"][:34], "grid": d.get("Grid Size", "")})
    v[d["Metric Name"]] = d["Metric Value"]
agg = collections.defaultdict(lambda: [0, 0.0])
for v in recs.values():
    if "gemm" not in v["name"]:
        continue
    a = agg[(v["name"], v["grid"])]
    a[0] += 1
    a[1] += float(v["gpu__time_duration.sum"].replace(",", "")) / 1e3
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{t / 1e3:9.2f} ms {n:5d} x {t / n:9.1f} us  {k[0]} {k[1]}")
