"""Per-kernel breakdown of decode iterations from an ncu launch list (csv of
gpu__time_duration.sum).  Iterations are delimited by decode_rows launches;
prints the mean per-iteration time of each kernel class and the total."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "ID"]
starts = [i for i, d in enumerate(data) if d["Kernel Name"].startswith("decode_rows")]
if len(starts) < 3:
    sys.exit("fewer than 3 decode iterations captured")
its = list(zip(starts[1:-1], starts[2:]))
agg = collections.defaultdict(float)
cnt = collections.defaultdict(int)
for a, b in its:
    for d in data[a:b]:
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")[:34] + " " + d["Grid Size"]
        agg[name] += float(d["Metric Value"].replace(",", "")) / 1000.0
        cnt[name] += 1
n = len(its)
tot = sum(agg.values()) / n
print(f"{n} iterations, {sum(cnt.values()) / n:.0f} kernels/iteration, {tot:.1f} us/iteration")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"{v / n:9.1f} us {100 * v / n / tot:5.1f}%  x{cnt[k] / n:5.1f}  {k}")
