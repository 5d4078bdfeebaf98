#!/usr/bin/env python
"""OPPO PPO-RLHF step benchmark on B200 (BASELINE.json metric).

Workload (configs[1]): 0.5B-shaped actor + 0.5B reward / critic / reference,
bf16, 256 prompts of 128 tokens per GPU, lognormal(5.0, 1.0) response lengths
capped at 1024, chunk 64, overcommit delta 26 (10%).  One step = refill ->
run_step (lockstep actor decode || streamed scorer prefill) -> select the
first B finishers -> PPO update (GAE, whitening, clipped loss, full-parameter
actor and critic update).  Reported next to the same binary with overlap disabled
(RunConfig::baseline(): delta 0, sequential scoring) and next to the
reference's own CPU path (oracle/_ref run_seed, toy policy) on the host cores.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

The PPO update trains every parameter of the actor and the critic
(train_heads=2: training forward + backward through all layers, SGD on fp32
masters), as the reference's toy_rlhf_step updates every policy parameter.
"""
import os

# K13 device-side chunk hand-off needs every kernel loaded before the step
# (a polling scorer kernel and a lazily loaded actor kernel deadlock); set
# before CUDA initialises in this process
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PPO samples/sec per step (overlap vs sequential) at 1/2/4/8 B200; roofline %"
CFG3_SMS, CFG4_SMS = 40, 32  # measured: cfg3 24/32/40/56 -> 62.5/66.4/67.1/65.3, cfg4 16/24/32/64 -> 8.3/8.4/8.3/7.1 samples/s
# scorer_sms: the fixed SM partition of the overlapped arm, measured per workload
CFG2 = dict(name="cfg2", actor="0.5b", scorer="0.5b", batch=256, prompt_len=128, mu=5.0,
            sigma=1.0, cap=1024, chunk=64, delta=26, scorer_sms=56)
# BASELINE configs[2] shape on one GPU: 1.5B actor + 0.5B scorers (chunk 64, 10% overcommit)
CFG3 = dict(name="cfg3", actor="1.5b", scorer="0.5b", batch=256, prompt_len=128, mu=5.0,
            sigma=1.0, cap=1024, chunk=64, delta=26, scorer_sms=CFG3_SMS)
# BASELINE configs[3] per GPU: 7B actor + 1.5B scorers, 512 prompts over 8 GPUs = 64 per GPU,
# LN(5.5, 1.0) cap 2048, 10% overcommit (6 per GPU)
CFG4 = dict(name="cfg4", actor="7b", scorer="1.5b", batch=64, prompt_len=128, mu=5.5,
            sigma=1.0, cap=2048, chunk=64, delta=6, scorer_sms=CFG4_SMS)
# BASELINE configs[4] per GPU: 7B actor, 4K max response, heavy long tail LN(6.0, 1.2) cap 4096,
# 256 prompts over 8 GPUs = 32 per GPU (KV + the 7B update's fp32 masters / gradients fit 180 GB),
# 10% overcommit (3 per GPU), chunk 128
CFG5 = dict(name="cfg5", actor="7b", scorer="1.5b", batch=32, prompt_len=128, mu=6.0,
            sigma=1.2, cap=4096, chunk=128, delta=3, scorer_sms=CFG4_SMS)
WORKLOADS = {}
TINY = dict(name="cfg1", actor="tiny", scorer="tiny", batch=8, prompt_len=8, mu=3.5, sigma=0.6,
            cap=64, chunk=16, delta=2)
WORKLOADS.update(cfg1=TINY, cfg2=CFG2, cfg3=CFG3, cfg4=CFG4, cfg5=CFG5)


def workload(args):
    """The --workload entry with the --chunk / --delta / --batch overrides."""
    wl = dict(WORKLOADS[args.workload])
    for k in ("chunk", "delta", "batch"):
        if getattr(args, k, None) is not None:
            wl[k] = getattr(args, k)
            wl["name"] += f" {k}={wl[k]}"
    return wl


def kv_bytes_per_token(shape):
    """K + V bytes (bf16) one token adds to a model's cache over all layers."""
    from paper_2509_25762_b200.engine import SHAPES
    d = SHAPES[shape]
    return 2 * d["n_layers"] * d["n_kv_heads"] * d["head_dim"] * 2


def peaks():
    """(HBM GB/s, bf16 TFLOP/s burst, bf16 TFLOP/s sustained, source)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1590.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, gpu=0):
        self.samples, self.proc, self.gpu = [], None, gpu

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# --------------------------------------------------------------- our arm
def host_prompts(ids, P, V, seed):
    """Synthetic prompt tokens on the host (the e2e path copies them in)."""
    out = []
    for i in ids:
        rng = np.random.default_rng([seed, int(i)])
        out.append(rng.integers(0, V, size=P, dtype=np.int32))
    return out


def run_arm(eng, wl, cfg, seed, steps, warmup, rank, world, dist):
    """The step loop in the engine's C++ host (oppo_run_seed_ex = driver.cpp:
    103-195 per rank, data parallel when world > 1): host prompts copied in
    at admission through the prompt-source hook, each step's record and
    ledger read back.  The per-step hook puts the warm-up boundary (device
    synchronize + barrier) before the timed steps.  Returns the timed steps."""
    import torch

    V = eng.cfg.actor.vocab
    P = cfg.prompt_len
    marks = {"prompts": [0] * (warmup + steps + 1)}
    state = {"step": 0}

    def prompt_fn(sid, plen):
        marks["prompts"][state["step"]] += plen * 4
        return host_prompts([sid], plen, V, 1234)[0]

    def on_step(rec):
        state["step"] = rec.step + 1
        if rec.step == warmup - 1:
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            marks["t0"] = time.perf_counter()
        return False

    if warmup == 0:
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        marks["t0"] = time.perf_counter()
    run_cfg = abi_copy(cfg)
    run_cfg.steps = warmup + steps
    recs, sel, leds = eng.run_seed_ex(run_cfg, seed, prompt_fn=prompt_fn, on_step=on_step)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    wall = time.perf_counter() - marks["t0"]
    if len(recs) != warmup + steps:
        raise RuntimeError(f"step loop ended after {len(recs)} steps")
    from paper_2509_25762_b200 import abi
    out = []
    for r, led in list(zip(recs, leds))[warmup:]:
        out.append(dict(samples=r.finished, step_us=led.step_us, update_us=r.update_us, loop_us=led.decode_loop_us,
                        decode_flops=led.decode_flops, prefill_flops=led.prefill_flops,
                        prefill_bytes=led.prefill_bytes, loop_kv_bytes=led.decode_kv_bytes,
                        loop_bytes=led.decode_weight_bytes + led.decode_kv_bytes, decode_us=led.decode_us,
                        score_us=led.score_us, iters=led.decode_iters, decode_tokens=led.decode_tokens,
                        prefill_tokens=led.prefill_tokens, launches=led.kernel_launches,
                        h2d=marks["prompts"][r.step] + r.finished * C.sizeof(abi.SeqState),
                        d2h=C.sizeof(abi.StepRecord) + C.sizeof(abi.Ledger) + int(r.batch_tokens) * 4 + r.finished * 4,
                        tokens=int(r.batch_tokens), reward=r.mean_reward, obj=r.ppo_loss,
                        util_actor=r.util_generation, util_scorer=r.util_scoring))
    return out, wall


def abi_copy(cfg):
    from paper_2509_25762_b200 import abi
    return abi.RunConfig.from_buffer_copy(cfg)


def abi_stats():
    from paper_2509_25762_b200 import abi
    return abi.PpoStats()


def workload_from_config(path):
    """A bench workload from a reference-schema JSON run config (+ our optional
    "model" / "gpu" blocks, paper_2509_25762_b200/config.py): the config's
    batch, prompt length, Delta range and controller, chunk size and length
    distribution drive the step loop; the metric stays BASELINE.json's."""
    from paper_2509_25762_b200 import abi
    from paper_2509_25762_b200 import config as K
    c = K.load_config(path, extended=True)
    if c["lengths"]["kind"] != abi.LEN_LOGNORMAL:
        raise K.ConfigError("bench --config needs lognormal lengths (the BASELINE workload shape)")
    model, gpu = c.get("model") or {}, c.get("gpu") or {}
    actor, scorer = model.get("actor", "0.5b"), model.get("reward", "0.5b")
    if not isinstance(actor, str) or not isinstance(scorer, str):
        raise K.ConfigError("bench --config takes engine shape names in model.actor / model.reward")
    rc = K.to_run_config(c)
    rc.mode, rc.steps = abi.RUN_TRAIN, 1000
    rc.carry_granularity = gpu.get("carry", abi.CARRY_TOKEN)
    rc.ppo.kl_coef, rc.ppo.whiten = gpu.get("kl_coef", 0.05), int(gpu.get("whiten", True))
    return dict(name=f"config {os.path.basename(path)} (fingerprint {K.task_fingerprint(c)})", actor=actor,
                scorer=scorer, batch=c["batch_size"], prompt_len=c["prompt_len"], mu=c["lengths"]["mu_log"],
                sigma=c["lengths"]["sigma_log"], cap=c["lengths"]["cap"], chunk=c["chunk_size"],
                delta=c["delta_max"], run_cfg=rc, scorer_sms=gpu.get("scorer_sms"))


def make_cfg(wl, baseline=False, ref_side=False):
    """The workload's RunConfig.  ref_side: built by the reference library
    (oracle/_ref) alone, so the reference arm never maps liboppo.so."""
    from paper_2509_25762_b200 import abi
    if ref_side:
        from oracle import ref as R
        default_config, base_fn = R.default_config, R.baseline_config
    else:
        from paper_2509_25762_b200 import scheduler as S
        default_config, base_fn = S.default_config, S.baseline
    if "run_cfg" in wl:
        cfg = abi.RunConfig.from_buffer_copy(wl["run_cfg"])
        return base_fn(cfg) if baseline else cfg
    cfg = default_config(
        mode=abi.RUN_TRAIN, steps=1000, batch_size=wl["batch"], prompt_len=wl["prompt_len"],
        delta_init=wl["delta"], delta_min=0, delta_max=wl["delta"], chunk_size=wl["chunk"],
        schedule_mode=abi.MODE_STREAMED, carry_granularity=abi.CARRY_TOKEN,
        lengths_kind=abi.LEN_LOGNORMAL, lengths_mu_log=wl["mu"], lengths_sigma_log=wl["sigma"],
        lengths_cap=wl["cap"], latency_decode_per_token=1, latency_prefill_per_token=0,
        latency_reward_residual=0, latency_placement=abi.PLACE_DISAGGREGATED,
        ppo_gamma=1.0, ppo_lambda=0.95, ppo_clip_epsilon=0.2, ppo_learning_rate=1e-3,
        ppo_value_learning_rate=1e-3, ppo_kl_coef=0.05, ppo_whiten=1)
    return base_fn(cfg) if baseline else cfg


def decode_roofline(recs, hbm_peak, peak_src, actor):
    """The dominant unit of the step: one actor decode iteration (a CUDA graph
    of ~7 launches per layer: RMSNorm, q|k|v GEMM, fused RoPE/KV-append/paged
    attention, O GEMM, RMSNorm, gate|up+SwiGLU GEMM, down GEMM, + lm_head /
    sampling), timed live with CUDA events on the actor stream over the timed
    steps' decode loops.  Algorithmic bytes per iteration (SURVEY 8d B_dec):
    the actor's weights once (non-embedding + lm_head) + per active row the KV
    positions it reads and the row it appends.  `traffic` is the ncu DRAM
    bytes of one iteration of the same build and actor shape
    (tools/capture_roofline.sh), at the captured row count nearest the step's
    mean active rows; its own algorithmic bytes are given beside it."""
    from paper_2509_25762_b200.engine import SHAPES
    loop_us = sum(r["loop_us"] for r in recs)
    loop_b = sum(r["loop_bytes"] for r in recs)
    iters = sum(r["iters"] for r in recs)
    if loop_us <= 0 or iters <= 0:
        return None
    ach = loop_b / (loop_us * 1e-6) / 1e9
    rows = sum(r["decode_tokens"] for r in recs) / iters
    out = {"kernel": f"actor decode iteration (CUDA graph: {SHAPES[actor]['n_layers']} layers + "
                     f"lm_head/sampling, {actor} actor, mean {rows:.0f} active rows)",
           "bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
           "frac": round(ach / hbm_peak, 4), "traffic": None,
           "algorithmic_bytes_per_launch": round(loop_b / iters),
           "avg_launch_us": round(loop_us / iters, 2),
           "peak_source": peak_src + " (MEASURED_PEAKS.json hbm_gbs)",
           "timing": "CUDA events on the actor stream around each step's decode loop"}
    caps = []
    for m in (16, 64, 128, 256):
        path = os.path.join(ROOT, "profiles", f"r02_decode_traffic_{actor}_M{m}.json")
        if os.path.exists(path):
            caps.append((abs(m - rows), m, path))
    if caps:
        _, m, path = min(caps)
        with open(path) as f:
            t = json.load(f)
        out["traffic"] = t["dram_bytes_per_iteration"]
        out["traffic_capture"] = {"rows": m, "file": os.path.relpath(path, ROOT),
                                  "algorithmic_bytes": t.get("algorithmic_bytes_per_iteration"),
                                  "traffic_over_algorithmic": t.get("traffic_over_algorithmic"),
                                  "source": t["source"]}
    return out


def step_roofline(recs, wl, hbm_peak, tf_sustained):
    """Step roofline: T_roof = max(F / peak_bf16, B / BW_HBM) over the
    step's algorithmic work -- actor decode (ledger: 2 P_dec + attention per
    sampled token; weights per iteration + KV), scorer prefill (ledger: linear
    + causal attention + the reference model's lm_head rows; weights per pass
    + KV), and the full-parameter update (6 P per training row for the actor
    and critic trunks, 6 V d per response token for the actor's lm_head;
    bytes: bf16 weights read twice, fp32 gradient written and read, fp32
    master read and written, bf16 weights rewritten = 22 B per parameter, plus
    the saved activations written once and read once).  Training attention is
    omitted (< 5% of the update's flops at these lengths).  frac = T_roof / T."""
    from paper_2509_25762_b200.engine import SHAPES
    a, c = SHAPES[wl["actor"]], SHAPES[wl["scorer"]]

    def nonemb(d):
        qkv = (d["n_heads"] + 2 * d["n_kv_heads"]) * d["head_dim"]
        return d["n_layers"] * (qkv * d["d_model"] + d["n_heads"] * d["head_dim"] * d["d_model"]
                                + 3 * d["d_model"] * d["d_ff"])

    def act_bytes(d):  # saved activations per training row (write + read), bf16 / fp32
        qkv = (d["n_heads"] + 2 * d["n_kv_heads"]) * d["head_dim"]
        per = 2 * d["d_model"] * 4 + 2 * d["d_model"] * 2 + qkv * 2 + d["n_heads"] * d["head_dim"] * 2 \
            + 3 * d["d_ff"] * 2
        return 2 * d["n_layers"] * per

    F = B = T = 0.0
    for r in recs:
        rows = r["tokens"] + r["samples"] * (wl["prompt_len"] - 1)
        f_tr = 6.0 * (nonemb(a) + nonemb(c)) * rows + 6.0 * a["vocab"] * a["d_model"] * r["tokens"]
        p_tr = nonemb(a) + nonemb(c) + a["vocab"] * a["d_model"] * (1 if a["tied"] else 2)
        b_tr = 22.0 * p_tr + rows * (act_bytes(a) + act_bytes(c))
        F += r["decode_flops"] + r["prefill_flops"] + f_tr
        B += r["loop_bytes"] + r["prefill_bytes"] + b_tr
        T += (r["step_us"] + r["update_us"]) * 1e-6
    t_f, t_b = F / (tf_sustained * 1e12), B / (hbm_peak * 1e9)
    t_roof = max(t_f, t_b)
    return {"flops_per_step": round(F / len(recs)), "bytes_per_step": round(B / len(recs)),
            "t_roof_ms": round(t_roof / len(recs) * 1e3, 2), "t_measured_ms": round(T / len(recs) * 1e3, 2),
            "bound": "tensor" if t_f >= t_b else "hbm", "frac": round(t_roof / T, 4),
            "peaks": {"bf16_tflops_sustained": tf_sustained, "hbm_gbs": hbm_peak}}


def gemm_microbench(hbm_peak):
    """Secondary: the decode gate|up GEMM alone at M=64 rows (the step's median
    batch), 24 distinct weight copies so weights stream from HBM."""
    from paper_2509_25762_b200._lib import lib
    M, N, K = 64, 2 * 4864, 896
    us = C.c_float()
    if lib().oppo_k_gemm_bench(M, N, K, 24, 240, 17, C.byref(us)) != 0:
        return None
    algo = N * K * 2 + M * K * 2 + M * (N // 2) * 2
    ach = algo / (us.value * 1e-6) / 1e9
    return {"kernel": "gemm_dec (swap-AB tcgen05+TMA) gate|up+SwiGLU, M=64 N=9728 K=896",
            "achieved": round(ach, 1), "unit": "GB/s", "frac": round(ach / hbm_peak, 4),
            "avg_launch_us": round(us.value, 3)}


def prefill_gemm_microbench(tf_peak):
    """The scorers' dominant kernel: the prefill gate|up GEMM (tcgen05 + TMA,
    128x256 tiles, SwiGLU epilogue) at an 8192-row pass, tensor roofline."""
    from paper_2509_25762_b200._lib import lib
    M, N, K = 8192, 2 * 4864, 896
    us = C.c_float()
    if lib().oppo_k_gemm_bench(M, N, K, 2, 50, 2, C.byref(us)) != 0:
        return None
    ach = 2.0 * M * N * K / (us.value * 1e-6) / 1e12
    return {"kernel": "gemm_bf16_tc<256> (tcgen05+TMA, 2 CTAs/SM) gate|up+SwiGLU, M=8192 N=9728 K=896",
            "bound": "tensor", "achieved": round(ach, 1), "unit": "TFLOP/s", "peak": tf_peak,
            "frac": round(ach / tf_peak, 4), "avg_launch_us": round(us.value, 3)}


def toy_reference(wl, budget_s=8.0):
    """The reference's own CPU path (oracle/_ref = /root/reference core compiled
    here): run_seed in train mode with its tabular toy policy (V=16) at this
    workload's B / delta / chunk / length distribution, one seed per host
    core.  Reported beside the neural port for scale (not the same workload)."""
    try:
        from oracle import ref as R
        if not R.available():
            return None
        from paper_2509_25762_b200 import scheduler as S
        cores = os.cpu_count() or 1
        cfg = make_cfg(wl, ref_side=True)
        S.set_field(cfg, "vocab", 16)
        S.set_field(cfg, "ppo_learning_rate", 0.1)
        S.set_field(cfg, "ppo_value_learning_rate", 0.2)
        cfg.carry_granularity = 0
        cfg.steps = 2
        t = time.perf_counter()
        R.run_seeds_parallel(cfg, list(range(1, cores + 1)))
        per = (time.perf_counter() - t) / 2
        cfg.steps = max(2, int(budget_s / max(per, 1e-3)))
        t = time.perf_counter()
        fin = R.run_seeds_parallel(cfg, list(range(1, cores + 1)))
        dt = time.perf_counter() - t
        return {"value": round(fin / dt, 1), "unit": "samples/s", "cores": cores, "kind": "reference",
                "sample": f"rlpipe::run_seed train mode (toy tabular policy V=16), B={wl['batch']}, "
                          f"delta={wl['delta']}, C={wl['chunk']}, LN({wl['mu']},{wl['sigma']}) cap "
                          f"{wl['cap']}, {cfg.steps} steps x {cores} seeds in {dt:.1f}s"}
    except Exception as ex:  # the baseline is reported, never required
        return {"value": None, "error": str(ex)[:200]}


def port_step_counts(wl, seed=7, steps=12):
    """Per-step counts of the workload for the CPU port: decode iterations per
    step from the reference's own run_seed (oracle/_ref, simulate mode, the
    lockstep latency model: one tick per decode iteration), and the token
    counts of a steady-state step (B samples, each response decoded once,
    each prompt + response prefilled once per scorer and trained once)."""
    from oracle import ref as R
    from paper_2509_25762_b200 import abi
    cfg = make_cfg(wl, ref_side=True)
    cfg.mode = abi.RUN_SIMULATE
    cfg.steps = steps
    cfg.carry_granularity = 0
    recs, _ = R.run_seed(cfg, seed)
    iters = float(np.mean([r.wall_ticks for r in recs[2:]]))
    lens = np.asarray(R.sample_lengths(cfg.lengths, seed, 100000), dtype=np.float64)
    B, P = wl["batch"], wl["prompt_len"]
    mean_len = lens.mean()
    dec_tokens = B * mean_len
    ctx = P + (lens * (lens + 1) / 2).sum() / lens.sum()  # mean context of a decoded token
    return dict(iters=iters, rows=dec_tokens / iters, ctx=ctx, prefill_tokens=B * (P + mean_len),
                train_rows=B * (P - 1 + mean_len), samples=B)


def cpu_port(wl, counts=None):
    """the same neural workload on the host cores -- the fp32
    all-cores numpy port of the engine's step (oracle/cpu_step.py: batched
    decode iteration, scorer prefill, training forward + backward), each
    timed on a bounded sample and projected to one step of this workload."""
    try:
        from oracle import cpu_step as P
        from paper_2509_25762_b200.engine import SHAPES
        c = counts or port_step_counts(wl)
        rows, ctx = max(1, round(c["rows"])), max(2, round(c["ctx"]))
        seq = int(min(wl["cap"], round(c["train_rows"] / c["samples"]))) + 1
        resp = max(1, seq - wl["prompt_len"])
        t = time.perf_counter()
        t_dec, t_pf, t_tr = P.measure(SHAPES[wl["actor"]], SHAPES[wl["scorer"]], rows, ctx, seq, resp)
        dt = time.perf_counter() - t
        step, v = P.project(t_dec, t_pf, t_tr, c["iters"], c["prefill_tokens"], c["train_rows"], c["samples"])
        return {"value": round(v, 5), "unit": "samples/s", "cores": P.cores(), "kind": "port",
                "sample": f"oracle/cpu_step.py fp32 numpy, BLAS on all cores: one {wl['actor']} decode iteration "
                          f"at {rows} rows x ctx {ctx} ({t_dec:.2f} s), {wl['scorer']} prefill of 2 x {seq} "
                          f"tokens ({t_pf * 1e3:.2f} ms/token), training fwd+bwd of {seq} rows "
                          f"({t_tr * 1e3:.2f} ms/row), measured in {dt:.1f} s; projected to a step of "
                          f"{c['iters']:.0f} iterations, 3 x {c['prefill_tokens']:.0f} prefill tokens, "
                          f"2 x {c['train_rows']:.0f} training rows = {step:.0f} s for {c['samples']} samples",
                "step_s": round(step, 1)}
    except Exception as ex:
        return {"value": None, "error": str(ex)[:200]}


def ours(args):
    import torch
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    dist = None
    if world > 1:
        import torch.distributed as td
        torch.cuda.set_device(local)
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = td
    torch.cuda.set_device(local)
    from paper_2509_25762_b200 import abi
    from paper_2509_25762_b200.engine import Engine, param_count, SHAPES, nccl_comm_from_torch
    comm = nccl_comm_from_torch(rank, world, local) if world > 1 else None

    wl = workload(args)
    if wl.get("train_rows"):
        os.environ.setdefault("OPPO_TRAIN_ROWS", str(wl["train_rows"]))
    hbm, tflops, tf_sust, peak_src = peaks()
    res = {}
    # overlap ablations: intra-step only = streamed scoring with
    # delta 0; inter-step only = overcommit with sequential (after-generation) scoring
    arms = [("oppo", False)] + ([] if args.no_sequential else [("sequential", True)])
    clocks = ClockSampler(local)
    with clocks:
        for name, base in arms:
            cfg = make_cfg(wl, base)
            if not base and args.overlap == "intra":
                cfg.delta_init = cfg.delta_min = cfg.delta_max = 0
            elif not base and args.overlap == "inter":
                cfg.schedule_mode = abi.MODE_SEQUENTIAL
            eng = Engine(wl["actor"], wl["scorer"], wl["scorer"], wl["scorer"], dtype=abi.DTYPE_BF16,
                         max_slots=wl["batch"] + wl["delta"] + 8, max_prompt_len=wl["prompt_len"],
                         max_response_len=wl["cap"], page_size=64, device=local,
                         carry=cfg.carry_granularity, train_heads=2, sample_seed=2 + rank,
                         weight_seed=1, scorer_sms=args.scorer_sms if not base else 0,
                         nccl_comm=comm, rank=rank, world=world)
            recs, wall = run_arm(eng, wl, cfg, 7, args.steps, args.warmup, rank, world, dist)
            eng.close()
            torch.cuda.empty_cache()
            dev_s = sum(r["step_us"] + r["update_us"] for r in recs) * 1e-6
            gen_s = sum(r["step_us"] for r in recs) * 1e-6
            samples = sum(r["samples"] for r in recs)
            t = torch.tensor([dev_s, gen_s, wall, float(samples)], dtype=torch.float64, device="cuda")
            if dist:
                mx = t.clone()
                dist.all_reduce(mx, op=dist.ReduceOp.MAX)
                sm = t.clone()
                dist.all_reduce(sm, op=dist.ReduceOp.SUM)
                dev_s, gen_s, wall = mx[0].item(), mx[1].item(), mx[2].item()
                samples = sm[3].item()
            res[name] = dict(recs=recs, dev_s=dev_s, gen_s=gen_s, wall=wall, samples=samples)
    if rank != 0:
        return
    o = res["oppo"]
    value = o["samples"] / o["dev_s"]
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(o["dev_s"] / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic prompts (host-generated tokens), random-init N(0,0.02) weights",
        "config": {"workload": f"{wl['name']}: {wl['actor']} actor + 3x {wl['scorer']} scorers "
                               f"(reward/critic/ref), B={wl['batch']}/GPU, prompt {wl['prompt_len']}, "
                               f"LN({wl['mu']},{wl['sigma']}) cap {wl['cap']}, chunk {wl['chunk']}, "
                               f"delta {wl['delta']}, token-granular carry"
                               + ("" if args.overlap == "both" else f", overlapped arm: {args.overlap}-step "
                                  "overlap only"),
                   "global_batch": wl["batch"] * world, "parallelism": f"dp{world}",
                   "params_per_model": param_count(SHAPES[wl["actor"]]),
                   "l2": "working set > L2 (4 models x ~1 GB bf16 weights + paged KV)",
                   "value_def": "samples / device time of (generation + scoring + PPO update)",
                   "sm_partition": f"scorers {args.scorer_sms} SMs | actor rest (green contexts)"
                                   if args.scorer_sms else "shared (stream priorities)"},
        "gen_score_samples_per_s": round(o["samples"] / o["gen_s"], 2),
    }
    if "sequential" in res:
        s = res["sequential"]
        line["sequential"] = {"value": round(s["samples"] / s["dev_s"], 2),
                              "gen_score_samples_per_s": round(s["samples"] / s["gen_s"], 2),
                              "ms_per_step": round(s["dev_s"] / args.steps * 1e3, 3)}
        line["speedup_vs_sequential"] = round(value / line["sequential"]["value"], 3)
        line["speedup_vs_sequential_gen_score"] = round(
            line["gen_score_samples_per_s"] / line["sequential"]["gen_score_samples_per_s"], 3)
    rec = o["recs"]
    line["e2e"] = {"value": round(o["samples"] / o["wall"], 2), "unit": "samples/s",
                   "h2d_bytes_per_step": int(np.mean([r["h2d"] for r in rec])),
                   "d2h_bytes_per_step": int(np.mean([r["d2h"] for r in rec]))}
    line["step_detail"] = {
        "decode_iters": int(np.mean([r["iters"] for r in rec])),
        "decode_ms": round(np.mean([r["decode_us"] for r in rec]) / 1e3, 2),
        "score_end_ms": round(np.mean([r["score_us"] for r in rec]) / 1e3, 2),
        "update_ms": round(np.mean([r["update_us"] for r in rec]) / 1e3, 2),
        "tokens_per_step": int(np.mean([r["tokens"] for r in rec])),
        "prefill_tokens_per_step": int(np.mean([r["prefill_tokens"] for r in rec])),
        # measured SM-partition utilization over the generation+scoring device time
        # (engine.cpp:225-233): actor decode loop, and the scorer waves' busy spans
        "util_actor_partition": round(float(np.mean([r["util_actor"] for r in rec])), 4),
        "util_scorer_partition": round(float(np.mean([r["util_scorer"] for r in rec])), 4),
    }
    line["roofline"] = decode_roofline(rec, hbm, peak_src, wl["actor"])
    line["step_roofline"] = step_roofline(rec, wl, hbm, tf_sust)
    line["kernels"] = {"decode_gemm_gate_up": gemm_microbench(hbm), "prefill_gemm_gate_up": prefill_gemm_microbench(tflops)}
    if not args.no_cpu:
        # the same neural workload on the host cores (the reference has no
        # neural path), with this run's own step counts; the reference's toy
        # tabular path beside it for scale (reported baselines, not targets)
        counts = dict(iters=float(np.mean([r["iters"] for r in rec])),
                      rows=float(np.sum([r["decode_tokens"] for r in rec]) / np.sum([r["iters"] for r in rec])),
                      ctx=float(np.sum([r["loop_kv_bytes"] for r in rec]) /
                                (kv_bytes_per_token(wl["actor"]) * np.sum([r["decode_tokens"] for r in rec]))),
                      prefill_tokens=float(np.mean([r["prefill_tokens"] for r in rec])),
                      train_rows=float(np.mean([r["tokens"] + r["samples"] * (wl["prompt_len"] - 1) for r in rec])),
                      samples=int(np.mean([r["samples"] for r in rec])))
        line["cpu_baseline"] = cpu_port(wl, counts)
        line["cpu_baseline"]["reference_toy"] = toy_reference(wl)
    else:
        line["cpu_baseline"] = None
    line["clocks"] = clocks.summary()
    line["gpu_launches"] = int(sum(r["launches"] for r in rec))
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def reference(args):
    """--impl reference: the CPU implementation of this workload on the host
    cores.  The reference has no neural path (its actor is a tabular toy,
    ppo.hpp:21-35), so each step is the all-cores port of the engine's step
    (oracle/cpu_step.py) on a bounded sample, projected to one step whose
    decode-iteration count comes from the reference's own run_seed
    (oracle/_ref, lockstep latency model); the reference's toy path at the
    same B / delta / chunk / lengths is reported beside it."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    wl = workload(args)
    try:
        from oracle import ref as R
        if not R.available():
            raise FileNotFoundError("oracle/_ref/librlpipe_ref.so not built")
        counts = port_step_counts(wl)
        for _ in range(args.warmup):
            cpu_port(wl, counts)
        vals, last = [], None
        for _ in range(args.steps):
            last = cpu_port(wl, counts)
            if last.get("value") is None:
                raise RuntimeError(last.get("error", "cpu port failed"))
            vals.append(last["value"])
        v = float(np.median(vals))
        step_s = wl["batch"] / v
        line = {"impl": "reference", "metric": METRIC, "value": round(v, 5), "unit": "samples/s",
                "n_gpus": int(os.environ.get("WORLD_SIZE", args.gpus)), "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 1),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (constant weights; timing only)",
                "config": {"workload": f"{wl['name']}: {wl['actor']} actor + 3x {wl['scorer']} scorers, "
                                       f"B={wl['batch']}, prompt {wl['prompt_len']}, LN({wl['mu']},{wl['sigma']}) "
                                       f"cap {wl['cap']}, chunk {wl['chunk']}, delta {wl['delta']}"},
                "cpu_baseline": {"value": round(v, 5), "unit": "samples/s", "cores": last["cores"],
                                 "kind": "port", "sample": last["sample"]},
                "reference_toy": toy_reference(wl),
                "e2e": {"value": round(v, 5), "unit": "samples/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
    except Exception as ex:
        line = {"impl": "reference", "unavailable": str(ex)[:200]}
    print(json.dumps(line), flush=True)


def free_port():
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: one process per GPU, launched here
    with the torchrun environment (RANK / LOCAL_RANK / WORLD_SIZE /
    MASTER_ADDR=127.0.0.1 / MASTER_PORT); rank 0's stdout is the JSON line."""
    port = free_port()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    codes = [p.wait() for p in procs]
    return max(codes, key=abs)


def dry_run_ranks(args):
    """--dry-run-ranks: the launch plumbing without a GPU: every rank joins a
    gloo group from the environment and rank 0 prints what it saw."""
    import torch
    import torch.distributed as td
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    td.init_process_group("gloo", rank=rank, world_size=world)
    t = torch.tensor([rank, int(os.environ.get("LOCAL_RANK", -1))], dtype=torch.int64)
    got = [torch.zeros_like(t) for _ in range(world)]
    td.all_gather(got, t)
    if rank == 0:
        print(json.dumps({"n_gpus": world, "ranks": [g.tolist() for g in got],
                          "global_batch": WORKLOADS[args.workload]["batch"] * world}), flush=True)
    td.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-sequential", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--scorer-sms", type=int, default=None,
                    help="fixed SM partition for the scorer stream in the overlapped arm (0: shared; "
                         "default: the workload's measured best)")
    ap.add_argument("--config", default=None,
                    help="reference-schema JSON run config (+ model/gpu blocks) instead of --workload")
    ap.add_argument("--dry-run-ranks", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--chunk", type=int, default=None, help="override the workload's chunk size")
    ap.add_argument("--delta", type=int, default=None, help="override the workload's overcommit delta")
    ap.add_argument("--batch", type=int, default=None, help="override the workload's per-GPU batch")
    ap.add_argument("--overlap", default="both", choices=["both", "intra", "inter"],
                    help="overlapped arm: both overlaps, intra-step only (delta 0), inter-step only "
                         "(sequential scoring)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        sys.exit(spawn_ranks(args.gpus))
    if args.dry_run_ranks:
        dry_run_ranks(args)
        return
    if args.config:
        wl = workload_from_config(args.config)
        WORKLOADS["config"] = wl
        args.workload = "config"
        if wl.get("scorer_sms") is not None and args.scorer_sms is None:
            args.scorer_sms = wl["scorer_sms"]
    if args.scorer_sms is None:
        args.scorer_sms = WORKLOADS[args.workload].get("scorer_sms", 56)
    if args.impl == "reference":
        reference(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
