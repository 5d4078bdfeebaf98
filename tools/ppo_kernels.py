"""HBM roofline of the per-token PPO kernels (K7 token_rewards, K8 gae_scan /
mc_returns, K9 moments, K10 ppo_clip) from an ncu csv of one PPO update
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
--kernel-name regex over those kernels; tools/update_profile.py).
Algorithmic bytes per token (fp32 engine arrays):
  token_rewards: old_lp, ref_lp in; reward, kl out          16 B
  gae_scan:      reward, value in; advantage, return out     16 B (+ one value per sequence)
  mc_returns:    return out                                   4 B
  moments:       advantage in                                 4 B
  ppo_clip:      new_lp, old_lp, advantage in; d obj out     16 B
Usage: ppo_kernels.py ncu.csv n_tokens hbm_peak_gbs"""
import collections
import csv
import json
import re
import sys

ALG = {"token_rewards": 16, "gae_scan": 16, "mc_returns": 4, "moments": 4, "ppo_clip": 16}
rows = list(csv.reader(open(sys.argv[1])))
n_tok, peak = float(sys.argv[2]), float(sys.argv[3])
hdr = next(r for r in rows if "Kernel Name" in r)
kern = collections.OrderedDict()
for r in rows:
    if len(r) != len(hdr) or r[0] == "ID":
        continue
    d = dict(zip(hdr, r))
    k = kern.setdefault(d["ID"], {"name": re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "")})
    v = float(d["Metric Value"].replace(",", ""))
    u = d.get("Metric Unit", "")
    if d["Metric Name"].startswith("dram__bytes"):
        k["dram"] = k.get("dram", 0.0) + v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    elif d["Metric Name"] == "gpu__time_duration.sum":
        k["us"] = v / 1e3 if u in ("nsecond", "ns") else v * (1e3 if u == "msecond" else 1.0)
agg = collections.defaultdict(lambda: {"launches": 0, "us": 0.0, "dram": 0.0})
for k in kern.values():
    base = next((b for b in ALG if b in k["name"]), None)
    if base is None:
        continue
    a = agg[base]
    a["launches"] += 1
    a["us"] += k.get("us", 0.0)
    a["dram"] += k.get("dram", 0.0)
out = {}
for b, a in agg.items():
    alg = ALG[b] * n_tok
    out[b] = {"launches": a["launches"], "total_us": round(a["us"], 2),
              "dram_bytes": round(a["dram"]), "algorithmic_bytes": round(alg),
              "dram_gbs": round(a["dram"] / (a["us"] * 1e-6) / 1e9, 1) if a["us"] else None,
              "algorithmic_gbs": round(alg / (a["us"] * 1e-6) / 1e9, 1) if a["us"] else None,
              "frac_of_hbm_peak": round(alg / (a["us"] * 1e-6) / 1e9 / peak, 4) if a["us"] else None}
print(json.dumps({"tokens": int(n_tok), "hbm_peak_gbs": peak, "kernels": out,
                  "note": "ncu serialises kernels and flushes caches per kernel (--cache-control all); "
                          "at ~1 MB per launch these kernels are launch/latency bound, not HBM bound"},
                 indent=1))
