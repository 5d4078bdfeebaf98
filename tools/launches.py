import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if 'Kernel Name' in r)
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != 'ID']
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    name = re.sub(r'\(.*', '', d['Kernel Name'])[:60] + " grid" + d['Grid Size']
    if 'gemm' not in name: name = re.sub(r' grid.*', '', name)
    v = float(d['Metric Value'].replace(',', '')) / 1000.0
    agg[name][0] += 1; agg[name][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{v[1]/1000:8.2f} ms {100*v[1]/tot:5.1f}% n={v[0]:6d} avg={v[1]/v[0]:8.2f}us  {k}")
print("total ms", tot/1000, "kernels", len(data))
