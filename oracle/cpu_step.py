"""TEST INFRASTRUCTURE ONLY — the all-cores CPU port of one OPPO step at a
bench workload: fp32 numpy with every matrix product on
BLAS (threaded over all host cores), used only by bench.py's cpu_baseline
leg and its --impl reference arm.  Never imported by the product.

The reference has no neural path (its actor is a tabular softmax,
ppo.hpp:21-35), so the same-workload CPU baseline is this port of the
engine's three phases, timed on bounded samples of the workload and
projected to the step from the GPU step's own counts:
  * actor decode: one batched decode iteration of R rows over a KV cache of
    `ctx` positions (per layer: RMSNorm, q|k|v + bias, RoPE, GQA attention
    over the cache, O + residual, RMSNorm, SwiGLU MLP + residual; final
    norm, lm_head, inverse-CDF sampling) -> seconds per iteration;
  * scorer prefill: causal forward of whole sequences through one scorer
    -> seconds per prefill token (x3 scorers);
  * PPO update: training forward + backward of one sequence through a trunk
    (RMSNorm / attention / SwiGLU backward, wgrad and dgrad products) plus
    the lm_head logits, softmax gradient and its two gradient products on
    the response rows -> seconds per training row (x2: actor and critic).
The model is the engine's (oracle/gpt_np.py states it in fp64 for parity);
weights are constants, whose values do not change the cost.
"""
import os
import time

import numpy as np

EPS = np.float32(1e-6)
F32 = np.float32


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class Port:
    def __init__(self, d):
        self.d = d
        D, V, F = d["d_model"], d["vocab"], d["d_ff"]
        self.qw = d["n_heads"] * d["head_dim"]
        self.qkv = self.qw + 2 * d["n_kv_heads"] * d["head_dim"]
        c = lambda *s: np.full(s, 0.01, dtype=F32)
        self.embed, self.lm_head = c(V, D), c(V, D)
        self.layers = [dict(wqkv=c(self.qkv, D), bqkv=c(self.qkv), wo=c(D, self.qw), wgu=c(2 * F, D),
                            wdown=c(D, F), g1=np.ones(D, F32), g2=np.ones(D, F32))
                       for _ in range(d["n_layers"])]
        self.gf = np.ones(D, F32)

    @staticmethod
    def rms(x, g):
        r = 1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + EPS)
        return x * r * g, r

    def rope_tab(self, pos):
        hd = self.d["head_dim"]
        inv = (1e6 ** (-2.0 * np.arange(hd // 2) / hd)).astype(F32)
        a = pos[:, None].astype(F32) * inv[None]
        return np.cos(a)[:, None], np.sin(a)[:, None]

    @staticmethod
    def rope(x, c, s, inv=False):
        h = x.shape[-1] // 2
        x1, x2 = x[..., :h], x[..., h:]
        if inv:
            s = -s
        return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], -1)

    # ---------------------------------------------------------- decode
    def decode_iteration(self, R, ctx, kv, rng, tok=None, return_logits=False):
        """One batched decode step at position ctx - 1 over kv[layer] = (K, V)
        caches [R, KV, >= ctx, hd] (the new row is written at ctx - 1)."""
        d = self.d
        H, KV, hd = d["n_heads"], d["n_kv_heads"], d["head_dim"]
        G = H // KV
        x = self.embed[rng.integers(0, d["vocab"], R) if tok is None else np.asarray(tok)]
        c, s = self.rope_tab(np.full(R, ctx - 1))
        for Lw, (kc, vc) in zip(self.layers, kv):
            h, _ = self.rms(x, Lw["g1"])
            qkv = h @ Lw["wqkv"].T + Lw["bqkv"]
            q = self.rope(qkv[:, :H * hd].reshape(R, H, hd), c, s).reshape(R, KV, G, hd)
            kc[:, :, ctx - 1] = self.rope(qkv[:, H * hd:(H + KV) * hd].reshape(R, KV, hd), c, s)
            vc[:, :, ctx - 1] = qkv[:, (H + KV) * hd:].reshape(R, KV, hd)
            sc = q @ kc[:, :, :ctx].transpose(0, 1, 3, 2) / np.sqrt(F32(hd))  # [R, KV, G, ctx]
            sc = np.exp(sc - sc.max(-1, keepdims=True))
            sc /= sc.sum(-1, keepdims=True)
            x = x + (sc @ vc[:, :, :ctx]).reshape(R, H * hd) @ Lw["wo"].T
            h2, _ = self.rms(x, Lw["g2"])
            gu = h2 @ Lw["wgu"].T
            g, u = gu[:, 0::2], gu[:, 1::2]
            x = x + ((g / (1.0 + np.exp(-g))) * u) @ Lw["wdown"].T
        hf, _ = self.rms(x, self.gf)
        lg = hf @ self.lm_head.T
        if return_logits:
            return lg
        p = np.exp(lg - lg.max(-1, keepdims=True))
        cdf = np.cumsum(p, -1)
        return (cdf < rng.random((R, 1), dtype=F32) * cdf[:, -1:]).sum(-1)

    # ---------------------------------------------------------- forward / backward
    def forward(self, tok, keep=False):
        d = self.d
        H, KV, hd = d["n_heads"], d["n_kv_heads"], d["head_dim"]
        G, T = H // KV, len(tok)
        x = self.embed[tok]
        c, s = self.rope_tab(np.arange(T))
        mask = np.triu(np.full((T, T), -np.inf, F32), 1)
        acts = []
        for Lw in self.layers:
            h1, r1 = self.rms(x, Lw["g1"])
            qkv = h1 @ Lw["wqkv"].T + Lw["bqkv"]
            q = self.rope(qkv[:, :H * hd].reshape(T, H, hd), c, s).transpose(1, 0, 2)  # [H, T, hd]
            k = self.rope(qkv[:, H * hd:(H + KV) * hd].reshape(T, KV, hd), c, s).transpose(1, 0, 2)
            v = qkv[:, (H + KV) * hd:].reshape(T, KV, hd).transpose(1, 0, 2)
            kk, vv = np.repeat(k, G, 0), np.repeat(v, G, 0)
            p = q @ kk.transpose(0, 2, 1) / np.sqrt(F32(hd)) + mask
            p = np.exp(p - p.max(-1, keepdims=True))
            p /= p.sum(-1, keepdims=True)
            o = (p @ vv).transpose(1, 0, 2).reshape(T, H * hd)
            xm = x + o @ Lw["wo"].T
            h2, r2 = self.rms(xm, Lw["g2"])
            gu = h2 @ Lw["wgu"].T
            g, u = gu[:, 0::2], gu[:, 1::2]
            sg = 1.0 / (1.0 + np.exp(-g))
            ff = g * sg * u
            if keep:
                acts.append(dict(x=x, h1=h1, r1=r1, q=q, kk=kk, vv=vv, p=p, o=o, xm=xm, h2=h2, r2=r2, g=g, u=u,
                                 sg=sg, ff=ff))
            x = xm + ff @ Lw["wdown"].T
        hf, rf = self.rms(x, self.gf)
        return hf, (acts, x, rf, c, s, tok)

    @staticmethod
    def rms_bwd(x, g, r, dy):
        xh = x * r
        dxh = dy * g
        return r * (dxh - xh * (dxh * xh).mean(-1, keepdims=True)), (dy * xh).sum(0)

    def backward(self, cache, d_hf):
        acts, xo, rf, c, s, tok = cache
        d = self.d
        H, KV, hd = d["n_heads"], d["n_kv_heads"], d["head_dim"]
        G, T = H // KV, d_hf.shape[0]
        dx, _ = self.rms_bwd(xo, self.gf, rf, d_hf)
        grads = []
        for Lw, a in zip(reversed(self.layers), reversed(acts)):
            gw = {"wdown": dx.T @ a["ff"]}
            dff = dx @ Lw["wdown"]
            dgu = np.empty((T, 2 * d["d_ff"]), F32)
            dgu[:, 1::2] = dff * a["g"] * a["sg"]
            dgu[:, 0::2] = dff * a["u"] * a["sg"] * (1.0 + a["g"] * (1.0 - a["sg"]))
            gw["wgu"] = dgu.T @ a["h2"]
            dxm, gw["g2"] = self.rms_bwd(a["xm"], Lw["g2"], a["r2"], dgu @ Lw["wgu"])
            dx = dx + dxm
            gw["wo"] = dx.T @ a["o"]
            do = (dx @ Lw["wo"]).reshape(T, H, hd).transpose(1, 0, 2)  # [H, T, hd]
            p = a["p"]
            dvv = p.transpose(0, 2, 1) @ do
            dp = do @ a["vv"].transpose(0, 2, 1)
            ds = p * (dp - (dp * p).sum(-1, keepdims=True)) / np.sqrt(F32(hd))
            dq = (ds @ a["kk"]).transpose(1, 0, 2)
            dk = (ds.transpose(0, 2, 1) @ a["q"]).reshape(KV, G, T, hd).sum(1).transpose(1, 0, 2)
            dv = dvv.reshape(KV, G, T, hd).sum(1).transpose(1, 0, 2)
            dqkv = np.concatenate([self.rope(dq, c, s, True).reshape(T, -1), self.rope(dk, c, s, True).reshape(T, -1),
                                   dv.reshape(T, -1)], 1)
            gw["bqkv"], gw["wqkv"] = dqkv.sum(0), dqkv.T @ a["h1"]
            dxi, gw["g1"] = self.rms_bwd(a["x"], Lw["g1"], a["r1"], dqkv @ Lw["wqkv"])
            dx = dx + dxi
            grads.append(gw)
        demb = np.zeros((256, d["d_model"]), F32)
        np.add.at(demb, tok % 256, dx)
        return grads


def measure(actor, scorer, rows, ctx, seq_len, resp_len, n_prefill_seqs=2, rng_seed=0):
    """(seconds per decode iteration at `rows` x `ctx`, per scorer prefill
    token, per training row), each from one bounded sample after a warm-up."""
    rng = np.random.default_rng(rng_seed)
    pa = Port(actor)
    KV, hd = actor["n_kv_heads"], actor["head_dim"]
    kv = [(np.zeros((rows, KV, ctx, hd), F32), np.zeros((rows, KV, ctx, hd), F32))
          for _ in range(actor["n_layers"])]
    pa.decode_iteration(min(rows, 16), ctx, [(k[:16], v[:16]) for k, v in kv], rng)  # warm
    t = time.perf_counter()
    pa.decode_iteration(rows, ctx, kv, rng)
    t_dec = time.perf_counter() - t
    del kv
    ps = pa if scorer == actor else Port(scorer)
    t = time.perf_counter()
    for _ in range(n_prefill_seqs):
        ps.forward(rng.integers(0, scorer["vocab"], seq_len))
    t_pf = (time.perf_counter() - t) / (n_prefill_seqs * seq_len)
    tok = rng.integers(0, actor["vocab"], seq_len)
    t = time.perf_counter()
    hf, cache = pa.forward(tok, keep=True)
    rr = hf[-resp_len:]
    lg = rr @ pa.lm_head.T
    gs = np.exp(lg - lg.max(-1, keepdims=True))
    gs /= -gs.sum(-1, keepdims=True)  # softmax gradient shape (values irrelevant)
    _ = gs.T @ rr  # lm_head wgrad
    d_hf = np.zeros_like(hf)
    d_hf[-resp_len:] = gs @ pa.lm_head  # dgrad
    pa.backward(cache, d_hf)
    t_tr = (time.perf_counter() - t) / seq_len
    return t_dec, t_pf, t_tr


def project(t_dec, t_pf, t_tr, iters, prefill_tokens, train_rows, samples):
    """Step seconds and samples/s of the CPU port for one step's counts:
    decode iterations, per-scorer prefill tokens (x3 scorers), training rows
    (x2 trained models)."""
    step = t_dec * iters + 3 * t_pf * prefill_tokens + 2 * t_tr * train_rows
    return step, samples / step
