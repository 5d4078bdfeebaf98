"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict


def main(path, top=40, by_grid=False):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0][:90]
        if by_grid and "gemm" in name:
            name += " grid" + d.get("Grid Size", "?")
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "nsecond")
        us = v / 1e3 if unit.startswith("n") else (v if unit.startswith("u") else v * 1e3)
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot / 1e3:.1f} ms over {sum(v[0] for v in agg.values())} launches")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{us / 1e3:9.2f} ms {100 * us / tot:5.1f}% {n:6d}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, len(sys.argv) > 3)
