"""Per-kernel share of the profiled region of an ncu launch list (csv of
gpu__time_duration.sum): kernels grouped by name (and grid for GEMMs),
serialized time and share; decode-path kernels flagged.  Shares, not
absolutes, compare with the live step (ncu serialises and flushes caches).
Usage: python tools/launch_share.py launches.csv"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "ID"]
agg, cnt = collections.defaultdict(float), collections.Counter()
for d in data:
    name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")[:40]
    us = float(d["Metric Value"].replace(",", "")) / 1e3
    agg[name] += us
    cnt[name] += 1
tot = sum(agg.values())
DEC = ("decode_rows", "gemm_dec", "attn_dec", "residual_rmsnorm", "lmhead_dec", "logits_combine")
dec = sum(v for k, v in agg.items() if any(x in k for x in DEC))
print(f"{len(data)} launches, {tot / 1e3:.1f} ms serialized; decode-path kernels {100 * dec / tot:.1f}%")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:30]:
    print(f"{v / 1e3:9.2f} ms {100 * v / tot:5.1f}%  x{cnt[k]:6d}  {k}")
