"""Diagnostics for tests/test_gpu_headline.py: per sampled sequence, the
engine's error against the bf16-rounding oracle and the fp64 oracle, and the
bf16-vs-fp64 oracle gap (how far bf16 rounding alone moves each quantity)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import test_gpu_headline as H  # noqa: E402
from oracle import gpt_np as N  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    run = H.run_cfg2(keep="all", weights=True)
    sel0 = run["log"][0]["selected"]
    by_len = sorted(sel0, key=lambda i: (run["rollouts"][i]["length"], i))
    picks = [by_len[0], by_len[len(by_len) // 4], by_len[len(by_len) // 2], by_len[-1]]
    P = 128
    rep = {i: {"length": run["rollouts"][i]["length"]} for i in picks}
    names = ["actor", "reward", "critic", "ref"]
    for mi, name in enumerate(names):
        dims, w = run["weights"][mi]
        for bfm in (True, False):
            m = N.GptNp(dims, w, bf16_mode=bfm)
            tag = "bf16" if bfm else "f64"
            for i in picks:
                ro = run["rollouts"][i]
                seq = np.concatenate([run["prompts"][i], ro["tokens"]]).astype(np.int64)
                L = ro["length"]
                r = rep[i]
                if name in ("actor", "ref"):
                    _, lg = m.forward(seq[:-1], rows=np.arange(P - 1, P + L - 1))
                    lp = H._logsm(lg)[np.arange(L), ro["tokens"][:L]]
                    got = ro["old_lp"] if name == "actor" else ro["ref_lp"]
                    r[f"{name}_lp_err_{tag}"] = float(np.abs(lp - got).max())
                    r[f"{name}_lp_mean_err_{tag}"] = float(np.abs(lp - got).mean())
                    if name == "actor" and bfm:
                        agree = checked = 0
                        margins = []
                        for j in range(L):
                            tok, _, mb, mi_ = O.sample_token(lg[j], O.token_key(H.SAMPLE_SEED, i, j + 1))
                            margins.append(min(mb, mi_))
                            if min(mb, mi_) > 1e-3:
                                checked += 1
                                agree += int(tok == ro["tokens"][j])
                        r["tokens_checked_1e-3"], r["tokens_agree_1e-3"] = checked, agree
                        r["min_margin"] = float(min(margins))
                    r[f"{name}_lp_vals_{tag}"] = [float(x) for x in lp[:3]]
                else:
                    hf, _ = m.forward(seq, logits=False)
                    if name == "critic":
                        v = hf[P - 1:P + L - 1] @ m.head
                        r[f"value_err_{tag}"] = float(np.abs(v - ro["values"]).max())
                        r[f"value_scale"] = float(np.abs(v).max())
                    else:
                        rw = float(hf[-1] @ m.head)
                        r[f"reward_{tag}"] = rw
                        r["reward_engine"] = float(ro["reward"])
            r2 = rep
            del m
    for i in picks:
        r = rep[i]
        r["reward_gap_bf16_vs_f64"] = abs(r["reward_bf16"] - r["reward_f64"])
        r["actor_lp_gap_bf16_vs_f64"] = None
    out = os.path.join(ROOT, "gpurun_out", "r02_headline_diag.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump({str(k): v for k, v in rep.items()}, f, indent=1)
    print(json.dumps({str(k): v for k, v in rep.items()}, indent=1))


if __name__ == "__main__":
    main()
