"""Per-kernel breakdown of the scorer wave(s) in an ncu launch list: every
launch after the last decode iteration (the last decode_rows + its ~200
iteration kernels) of the first run_step."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "ID"]
starts = [i for i, d in enumerate(data) if d["Kernel Name"].startswith("decode_rows")]
# end of the first step's decode loop: the first gap in consecutive decode_rows spacing
per = starts[1] - starts[0]
last = starts[0]
for a, b in zip(starts, starts[1:]):
    if b - a != per:
        break
    last = b
i0 = last + per
i1 = next((i for i in range(i0, len(data)) if data[i]["Kernel Name"].startswith("decode_rows")), len(data))
agg = collections.defaultdict(float)
cnt = collections.defaultdict(int)
for d in data[i0:i1]:
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")[:40]
    if "gemm" in name:
        name += " " + d["Grid Size"]
    agg[name] += float(d["Metric Value"].replace(",", "")) / 1000.0
    cnt[name] += 1
tot = sum(agg.values())
print(f"scorer wave: {i1 - i0} launches, {tot / 1000:.2f} ms serialized")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:25]:
    print(f"{v / 1000:8.2f} ms {100 * v / tot:5.1f}%  x{cnt[k]:5d}  {k}")
