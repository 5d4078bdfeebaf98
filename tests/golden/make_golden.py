"""Generates tests/golden/reference_vectors.json from the COMPILED REFERENCE
(oracle/_ref/librlpipe_ref.so, built from /root/reference/proj/core by
oracle/Makefile).  Run in the build container:  python tests/golden/make_golden.py

The fixtures pin (a) the reference's RNG/length streams, (b) build_schedule,
run_step under the lockstep latency model, select_finished, the Delta
controllers and the tuner, (c) whole run_seed decision traces, and (d) the
fp64 PPO math (compute_gae, clipped_objective, clipped_objective_grad,
rollout, toy_rlhf_step).  The GPU box has no /root/reference, so tests read
these vectors instead of the live reference there.
"""
import ctypes as C
import json
import os
import random
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle import ref as R  # noqa: E402
from paper_2509_25762_b200 import abi  # noqa: E402
from paper_2509_25762_b200 import scheduler as S  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "reference_vectors.json")


def lockstep(**kw):
    base = dict(latency_decode_per_token=1, latency_prefill_per_token=0,
                latency_reward_residual=0, latency_chunk_switch_cost=0,
                latency_transfer_per_chunk=0, latency_placement=abi.PLACE_DISAGGREGATED)
    base.update(kw)
    return S.default_config(**base)


def cfg_dict(cfg):
    d = {}
    for name, _ in cfg._fields_:
        v = getattr(cfg, name)
        if name == "chunk_candidates":
            d[name] = list(v)[:cfg.n_candidates]
        elif isinstance(v, C.Structure):
            sub = {}
            for n2, _ in v._fields_:
                x = getattr(v, n2)
                sub[n2] = list(x) if hasattr(x, "__len__") else x
            d[name] = sub
        else:
            d[name] = v
    return d


def random_states(rng, n, chunk):
    out = []
    for i in range(n):
        L = rng.randint(1, 80)
        g = rng.choice([0, 0, rng.randint(0, L)])
        if rng.random() < 0.5 and g > 0:
            g = (g // chunk) * chunk
        p = rng.randint(0, g) if g else 0
        out.append(dict(id=i * 3 + rng.randint(0, 2), prompt_len=rng.randint(1, 8),
                        target_len=L, generated=g, prefilled_tokens=p,
                        chunks_emitted=(g + chunk - 1) // chunk,
                        chunks_prefilled=(p + chunk - 1) // chunk if p else 0))
    # unique ids
    for i, s in enumerate(out):
        s["id"] = i * 3 + (s["id"] % 3)
    return out


def main():
    g = {"source": "oracle/_ref/librlpipe_ref.so (reference core @ /root/reference/proj/core)"}
    g["rng"] = {
        "lengths_u64": [str(x) for x in R.rng_draws(1, "lengths", 8)],
        "lengths_uniform01": R.rng_draws(1, "lengths", 8, "uniform01"),
        "lengths_normal": R.rng_draws(1, "lengths", 9, "normal"),
        "ppo_u64": [str(x) for x in R.rng_draws(1, "ppo", 4)],
        "seed_12345_prompt_u64": [str(x) for x in R.rng_draws(12345, "prompt", 4)],
    }
    dists = []
    for kind, kw in [
        (abi.LEN_LOGNORMAL, dict(mu_log=5.0, sigma_log=0.8, cap=4096)),
        (abi.LEN_LOGNORMAL, dict(mu_log=5.0, sigma_log=1.0, cap=1024)),
        (abi.LEN_LOGNORMAL, dict(mu_log=5.5, sigma_log=1.3, cap=4096)),
        (abi.LEN_LOGNORMAL, dict(mu_log=3.5, sigma_log=0.6, cap=64)),
        (abi.LEN_TWO_POINT, dict(fast_len=64, slow_len=128, p_slow=0.1, cap=4096)),
        (abi.LEN_EMPIRICAL, dict(cap=100, table=[(10, 1.0), (50, 2.5), (100, 0.5)])),
    ]:
        d = abi.LengthDist()
        d.kind = kind
        for k, v in kw.items():
            if k == "table":
                d.table_n = len(v)
                for i, (ln, w) in enumerate(v):
                    d.table_len[i], d.table_w[i] = ln, w
            else:
                setattr(d, k, v)
        for seed in (1, 7):
            dists.append({"kind": kind, "params": kw, "seed": seed,
                          "draws": R.sample_lengths(d, seed, 200)})
    g["lengths"] = dists

    rng = random.Random(2024)
    steps = []
    for trial in range(60):
        chunk = rng.choice([1, 3, 8, 16, 64])
        n = rng.randint(1, 12)
        states = random_states(rng, n, chunk)
        arr = S.seq_array(states)
        mode = rng.choice([0, 1])
        stop = rng.choice([0, 1, rng.randint(1, n), n, n + 2])
        sched = R.build_schedule(arr, n, chunk, mode)
        outs, led = R.run_step(arr, n, chunk, mode, R.lockstep_latency(), stop)
        steps.append({"states": states, "chunk": chunk, "mode": mode, "stop_after": stop,
                      "schedule": sched, "outcomes": [o.as_tuple() for o in outs],
                      "ledger": [led.wall, led.busy_generation, led.busy_scoring,
                                 led.work_generation, led.work_scoring]})
    g["lockstep_steps"] = steps

    ctl = []
    for trial in range(40):
        mode = rng.choice([abi.DELTA_ALG1, abi.DELTA_EQ4])
        w = rng.randint(1, 6)
        hist = [rng.uniform(-1, 1) if rng.random() < 0.8 else 0.5 for _ in range(rng.randint(0, 20))]
        delta = rng.randint(0, 12)
        h = (C.c_double * max(1, len(hist)))(*hist)
        nh, nd, hs, st = C.c_int32(len(hist)), C.c_int32(), C.c_int32(), C.c_double()
        R.rcheck(R.ref().ref_delta_update(mode, w, 0, 12, rng.randint(1, 3), rng.randint(1, 3),
                                          h, C.byref(nh), delta, C.byref(nd), C.byref(hs),
                                          C.byref(st)))
        ctl.append({"mode": mode, "window": w, "hist": hist, "delta": delta,
                    "inc_dec": None, "new_delta": nd.value, "has_stat": hs.value,
                    "stat": st.value, "hist_after": list(h[:nh.value])})
    g["controller"] = ctl

    runs = []
    specs = [
        ("appendix_a_cfg1", lockstep(steps=6, batch_size=8, prompt_len=8, delta_init=2,
                                     delta_max=2, chunk_size=16, lengths_kind=abi.LEN_LOGNORMAL,
                                     lengths_mu_log=3.5, lengths_sigma_log=0.6, lengths_cap=64), 1),
        ("cfg2_shape", lockstep(steps=12, batch_size=256, prompt_len=128, delta_init=26,
                                delta_max=26, chunk_size=64, lengths_kind=abi.LEN_LOGNORMAL,
                                lengths_mu_log=5.0, lengths_sigma_log=1.0, lengths_cap=1024), 3),
        ("cfg4_shape_rank", lockstep(steps=8, batch_size=64, prompt_len=128, delta_init=6,
                                     delta_max=13, chunk_size=64, controller=abi.DELTA_ALG1,
                                     window=2, proxy_kind=1, lengths_kind=abi.LEN_LOGNORMAL,
                                     lengths_mu_log=5.5, lengths_sigma_log=1.0,
                                     lengths_cap=2048), 2),
        ("tie_case", lockstep(steps=5, batch_size=2, prompt_len=1, delta_init=2, delta_max=2,
                              chunk_size=16, lengths_kind=abi.LEN_TWO_POINT, lengths_fast_len=17,
                              lengths_slow_len=40, lengths_p_slow=0.3, lengths_cap=64), 5),
        ("tuner", lockstep(steps=12, batch_size=16, prompt_len=4, delta_init=4, delta_max=4,
                           chunk_size=16, tune_chunks=1, chunk_candidates=[8, 16, 32],
                           retune_period=5, lengths_kind=abi.LEN_LOGNORMAL, lengths_mu_log=4.0,
                           lengths_sigma_log=0.9, lengths_cap=256), 9),
        ("eq4", lockstep(steps=20, batch_size=8, prompt_len=4, delta_init=3, delta_max=8,
                         chunk_size=8, controller=abi.DELTA_EQ4, window=3, proxy_kind=1,
                         proxy_ramp_steps=10, lengths_kind=abi.LEN_LOGNORMAL, lengths_mu_log=3.0,
                         lengths_sigma_log=0.8, lengths_cap=128), 11),
    ]
    base_specs = [(n + "_baseline", S.baseline(c), s) for n, c, s in specs[:3]]
    for name, cfg, seed in specs + base_specs:
        recs, sel, _ = R.trace_seed(cfg, seed)
        official, _ = R.run_seed(cfg, seed)
        assert [(r.wall_ticks, r.finished, r.deferred, r.delta) for r in recs] == \
               [(r.wall_ticks, r.finished, r.deferred, r.delta) for r in official], name
        runs.append({"name": name, "seed": seed, "config": cfg_dict(cfg),
                     "records": [[r.step, r.wall_ticks, r.finished, r.deferred, r.delta,
                                  r.has_controller_stat, r.controller_stat, r.mean_reward,
                                  r.util_generation, r.util_scoring, r.max_deferrals]
                                 for r in recs],
                     "selected": sel})
    g["runs"] = runs

    # ------------------------------------------------------------ PPO fp64
    L = R.ref()
    gae = []
    for trial in range(30):
        T = rng.randint(1, 40)
        rw = [rng.gauss(0, 1) for _ in range(T)]
        vals = [rng.gauss(0, 1) for _ in range(T + 1)]
        gm, lm = rng.random(), rng.random()
        out = (C.c_double * T)()
        R.rcheck(L.ref_compute_gae((C.c_double * T)(*rw), (C.c_double * (T + 1))(*vals), T, gm,
                                   lm, out))
        gae.append({"rewards": rw, "values": vals, "gamma": gm, "lambda": lm, "adv": list(out)})
    g["gae"] = gae

    clip = []
    for trial in range(20):
        vocab = rng.randint(2, 8)
        theta = [rng.gauss(0, 1) for _ in range((vocab + 1) * vocab)]
        nseq = rng.randint(1, 6)
        lens = [rng.randint(1, 12) for _ in range(nseq)]
        offs = [0]
        for ln in lens:
            offs.append(offs[-1] + ln)
        toks = [rng.randint(0, vocab - 1) for _ in range(offs[-1])]
        old = [-3.0 * rng.random() for _ in range(offs[-1])]
        vals = [rng.gauss(0, 1) for _ in range(offs[-1] + nseq)]
        rews = [rng.gauss(0, 1) for _ in range(nseq)]
        gm, lm, eps = rng.random(), rng.random(), rng.choice([0.1, 0.2, 0.3])
        obj = C.c_double()
        grad = (C.c_double * ((vocab + 1) * vocab))()
        D = C.c_double
        R.rcheck(L.ref_clipped_objective(vocab, (D * len(theta))(*theta), nseq,
                                         (C.c_int32 * len(offs))(*offs),
                                         (C.c_int32 * len(toks))(*toks), (D * len(old))(*old),
                                         (D * len(vals))(*vals), (D * nseq)(*rews), gm, lm, eps,
                                         C.byref(obj), grad))
        # per-token policy log-probs of the taken tokens (the GPU kernels' input)
        new_lp = []
        for i in range(nseq):
            prev = 0
            for t in range(offs[i], offs[i + 1]):
                lp = (D * vocab)()
                R.rcheck(L.ref_policy_logprobs(vocab, (D * len(theta))(*theta), prev, lp))
                new_lp.append(lp[toks[t]])
                prev = toks[t] + 1
        clip.append({"vocab": vocab, "theta": theta, "offsets": offs, "tokens": toks,
                     "old_lp": old, "values": vals, "rewards": rews, "gamma": gm, "lambda": lm,
                     "eps": eps, "objective": obj.value, "grad": list(grad), "new_lp": new_lp})
    g["clipped"] = clip

    # toy rollout (Appendix A) and one toy_rlhf_step
    D = C.c_double
    lens = [12, 5, 9]
    toks = (C.c_int32 * sum(lens))()
    olp = (D * sum(lens))()
    rw = (D * 3)()
    R.rcheck(L.ref_rollouts(16, None, 0, 1.0, 0.0, 1, 3, (C.c_int32 * 3)(*lens), toks, olp, rw))
    g["toy_rollout"] = {"vocab": 16, "seed": 1, "lengths": lens, "tokens": list(toks),
                        "old_lp": list(olp), "rewards": list(rw)}

    with open(OUT, "w") as f:
        json.dump(g, f, indent=0)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
