"""DRAM traffic and duration of one actor decode iteration from an ncu csv
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum).
Iterations are delimited by decode_rows launches; windows whose kernel count
differs from the most common one (e.g. a scorer wave between steps) are
dropped.  Prints a JSON summary (committed under profiles/)."""
import collections
import csv
import json
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if "Kernel Name" in r)
recs = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "ID"]
kern = collections.OrderedDict()
for d in recs:
    k = kern.setdefault(d["ID"], {"name": d["Kernel Name"], "grid": d["Grid Size"]})
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "")
    if d["Metric Name"].startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        k["dram"] = k.get("dram", 0.0) + v * scale
    elif d["Metric Name"] == "gpu__time_duration.sum":
        k["us"] = v / 1000.0 if unit in ("nsecond", "ns") else v * (1e3 if unit == "msecond" else 1.0)
ks = list(kern.values())
starts = [i for i, k in enumerate(ks) if k["name"].startswith("decode_rows")]
wins = [ks[a:b] for a, b in zip(starts, starts[1:])]
if not wins and starts:  # a single captured iteration: up to the end of the list
    wins = [ks[starts[0]:]]
mode = collections.Counter(len(w) for w in wins).most_common(1)[0][0]
wins = [w for w in wins if len(w) == mode]
dram = [sum(k.get("dram", 0.0) for k in w) for w in wins]
us = [sum(k.get("us", 0.0) for k in w) for w in wins]
by = collections.defaultdict(float)
for w in wins:
    for k in w:
        by[re.sub(r"\(.*", "", k["name"]).replace("void ", "")[:40]] += k.get("dram", 0.0) / len(wins)
out = {"iterations": len(wins), "kernels_per_iteration": mode,
       "dram_bytes_per_iteration": round(sum(dram) / len(dram)),
       "serialized_kernel_us_per_iteration": round(sum(us) / len(us), 1),
       "dram_bytes_by_kernel": {k: round(v) for k, v in sorted(by.items(), key=lambda kv: -kv[1])},
       "source": sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]}
if len(sys.argv) > 3:  # algorithmic bytes of one iteration of the captured run (decode_iter.py)
    out["algorithmic_bytes_per_iteration"] = round(float(sys.argv[3]))
    out["traffic_over_algorithmic"] = round(out["dram_bytes_per_iteration"] / float(sys.argv[3]), 3)
print(json.dumps(out, indent=1))
