"""TEST INFRASTRUCTURE ONLY — vectorised numpy restatement of the engine's
Qwen2-style decoder (the same model as oracle_gpt_forward in oppo_oracle.c,
cross-checked against it in tests/test_oracle.py), used where the scalar C
forward is too slow: full-depth 0.5B parity checks at the bench shape, the
fp64 backward that pins the full-parameter PPO update, and the all-cores CPU
baseline of bench.py.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import it.

Model (no reference counterpart — the reference's actor is a
tabular softmax, ppo.hpp:21-35): RMSNorm (eps 1e-6), q|k|v projection with
bias, rotate-half RoPE (theta 1e6) at the token's position in its sequence,
causal GQA attention, O projection + residual, RMSNorm, SwiGLU over
interleaved (gate_i, up_i) rows, down projection + residual, final RMSNorm,
lm_head (or a scalar head for the reward / critic).

bf16=True rounds activations to bf16 at the points where the engine stores
them in bf16 (normed rows, q|k|v + bias, RoPE'd q/k, attention weights fed
to P.V, attention output, SwiGLU output), everything else in fp64, so the
comparison with the bf16 engine measures accumulation-order noise only.
"""
import numpy as np

EPS = 1e-6
THETA = 1e6


def bf16(x):
    """Round to the nearest bf16 (ties to even), returned as float64."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def rope_tables(T, hd, pos0=0):
    half = hd // 2
    inv = THETA ** (-2.0 * np.arange(half) / hd)
    ang = (pos0 + np.arange(T))[:, None] * inv[None, :]
    return np.cos(ang), np.sin(ang)


def rope(x, cs, sn):
    """x [T, heads, hd] rotate-half."""
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    c, s = cs[:, None, :], sn[:, None, :]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def rope_bwd(dy, cs, sn):
    """Transpose of rope (rotation by -angle)."""
    half = dy.shape[-1] // 2
    d1, d2 = dy[..., :half], dy[..., half:]
    c, s = cs[:, None, :], sn[:, None, :]
    return np.concatenate([d1 * c + d2 * s, d2 * c - d1 * s], axis=-1)


class GptNp:
    """fp64 (optionally bf16-rounded) forward / backward of one model.

    w: the engine's weight export (engine.Engine.export_weights): embed [V,d],
    lm_head [V,d], final_norm [d], per layer ln1 [d], wqkv [qkv,d], bqkv
    [qkv], wo [d,H hd], ln2 [d], wgu [2F,d] (interleaved), wdown [d,F]."""

    def __init__(self, dims, w, bf16_mode=False, dtype=np.float64):
        self.dims, self.bf = dims, bf16_mode
        self.dt = dtype
        D, V, F = dims["d_model"], dims["vocab"], dims["d_ff"]
        qw = dims["n_heads"] * dims["head_dim"]
        qkv = qw + 2 * dims["n_kv_heads"] * dims["head_dim"]
        cv = lambda a, *shape: np.asarray(a, dtype=dtype).reshape(shape)  # exports are flat
        self.embed = cv(w["embed"], V, D)
        self.lm_head = cv(w["lm_head"], V, D)
        self.final_norm = cv(w["final_norm"], D)
        self.head = None if w.get("head") is None else cv(w["head"], D)
        L = dims["n_layers"]
        self.layers = [dict(ln1=cv(w["ln1"][l], D), wqkv=cv(w["wqkv"][l], qkv, D), bqkv=cv(w["bqkv"][l], qkv),
                            wo=cv(w["wo"][l], D, qw), ln2=cv(w["ln2"][l], D), wgu=cv(w["wgu"][l], 2 * F, D),
                            wdown=cv(w["wdown"][l], D, F)) for l in range(L)]

    def _r(self, x):
        return bf16(x) if self.bf else x

    @staticmethod
    def _rms(x, g):
        r = 1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + EPS)
        return x * r * g, r

    def forward(self, tokens, logits=True, rows=None, keep=False):
        """tokens [T] -> (final normed hidden [T,d], logits [len(rows) or T, V] or None).
        keep=True also returns the per-layer activations for backward()."""
        d = self.dims
        H, KV, hd, F = d["n_heads"], d["n_kv_heads"], d["head_dim"], d["d_ff"]
        G = H // KV
        tok = np.asarray(tokens, dtype=np.int64)
        T = len(tok)
        x = self.embed[tok].copy()
        cs, sn = rope_tables(T, hd)
        mask = np.triu(np.full((T, T), -np.inf), 1)
        acts = []
        for Lw in self.layers:
            a = dict(x_in=x.copy())
            h, r1 = self._rms(x, Lw["ln1"])
            h = self._r(h)
            qkv = self._r(h @ Lw["wqkv"].T + Lw["bqkv"])
            q = qkv[:, :H * hd].reshape(T, H, hd)
            k = qkv[:, H * hd:(H + KV) * hd].reshape(T, KV, hd)
            v = qkv[:, (H + KV) * hd:].reshape(T, KV, hd)
            q = self._r(rope(q, cs, sn))
            k = self._r(rope(k, cs, sn))
            kk = np.repeat(k, G, axis=1)  # [T, H, hd]
            vv = np.repeat(v, G, axis=1)
            s = np.einsum("thd,shd->hts", q, kk) / np.sqrt(hd) + mask[None]
            m = s.max(-1, keepdims=True)
            e = np.exp(s - m)
            z = e.sum(-1, keepdims=True)
            if self.bf:
                o = np.einsum("hts,shd->thd", bf16(e), vv) / np.transpose(z, (1, 0, 2))
            else:
                o = np.einsum("hts,shd->thd", e / z, vv)
            o = self._r(o.reshape(T, H * hd))
            x = x + o @ Lw["wo"].T
            a.update(h1=h, r1=r1, q=q, k=k, v=v, p=e / z, o=o, x_mid=x.copy())
            h2, r2 = self._rms(x, Lw["ln2"])
            h2 = self._r(h2)
            gu = h2 @ Lw["wgu"].T
            g, u = gu[:, 0::2], gu[:, 1::2]
            sg = 1.0 / (1.0 + np.exp(-g))
            ff = self._r(g * sg * u)
            x = x + ff @ Lw["wdown"].T
            a.update(h2=h2, r2=r2, gu=gu, ff=ff)
            if keep:
                acts.append(a)
        hf, rf = self._rms(x, self.final_norm)
        hf = self._r(hf)
        lg = None
        if logits:
            src = hf if rows is None else hf[np.asarray(rows)]
            lg = src @ self.lm_head.T
        if keep:
            return hf, lg, dict(layers=acts, x_out=x, rf=rf, cs=cs, sn=sn, tok=tok)
        return hf, lg

    def backward(self, cache, d_hf):
        """d_hf [T, d] = dLoss/d(final normed hidden) -> dict of parameter
        gradients (same names / layouts as the weight export, fp64) except the
        lm_head / head terms, which the caller adds (they need the logits)."""
        d = self.dims
        H, KV, hd = d["n_heads"], d["n_kv_heads"], d["head_dim"]
        G = H // KV
        T = d_hf.shape[0]
        cs, sn = cache["cs"], cache["sn"]
        grads = {k: [None] * len(self.layers) for k in ("ln1", "wqkv", "bqkv", "wo", "ln2", "wgu", "wdown")}
        dx, dg = self._rms_bwd(cache["x_out"], self.final_norm, cache["rf"], d_hf)
        grads["final_norm"] = dg
        scale = 1.0 / np.sqrt(hd)
        for l in range(len(self.layers) - 1, -1, -1):
            Lw, a = self.layers[l], cache["layers"][l]
            # down + SwiGLU
            grads["wdown"][l] = dx.T @ a["ff"]
            dff = dx @ Lw["wdown"]
            g, u = a["gu"][:, 0::2], a["gu"][:, 1::2]
            sg = 1.0 / (1.0 + np.exp(-g))
            dgu = np.empty_like(a["gu"])
            dgu[:, 1::2] = dff * g * sg
            dgu[:, 0::2] = dff * u * sg * (1.0 + g * (1.0 - sg))
            grads["wgu"][l] = dgu.T @ a["h2"]
            dh2 = dgu @ Lw["wgu"]
            dxm, grads["ln2"][l] = self._rms_bwd(a["x_mid"], Lw["ln2"], a["r2"], dh2)
            dx = dx + dxm
            # O projection + attention
            grads["wo"][l] = dx.T @ a["o"]
            do = (dx @ Lw["wo"]).reshape(T, H, hd)
            p = a["p"]  # [H, T, S]
            kk = np.repeat(a["k"], G, axis=1)
            vv = np.repeat(a["v"], G, axis=1)
            dvv = np.einsum("hts,thd->shd", p, do)
            dp = np.einsum("thd,shd->hts", do, vv)
            ds = p * (dp - (dp * p).sum(-1, keepdims=True))
            dq = np.einsum("hts,shd->thd", ds, kk) * scale
            dkk = np.einsum("hts,thd->shd", ds, a["q"]) * scale
            dk = dkk.reshape(T, KV, G, hd).sum(2)
            dv = dvv.reshape(T, KV, G, hd).sum(2)
            dq = rope_bwd(dq, cs, sn)
            dk = rope_bwd(dk, cs, sn)
            dqkv = np.concatenate([dq.reshape(T, -1), dk.reshape(T, -1), dv.reshape(T, -1)], axis=1)
            grads["bqkv"][l] = dqkv.sum(0)
            grads["wqkv"][l] = dqkv.T @ a["h1"]
            dh1 = dqkv @ Lw["wqkv"]
            dxi, grads["ln1"][l] = self._rms_bwd(a["x_in"], Lw["ln1"], a["r1"], dh1)
            dx = dx + dxi
        demb = np.zeros_like(self.embed)
        np.add.at(demb, cache["tok"], dx)
        grads["embed"] = demb
        return grads

    @staticmethod
    def _rms_bwd(x, g, r, dy):
        """y = x * r * g, r = (mean(x^2) + eps)^-1/2 -> (dx, dg)."""
        xh = x * r
        dg = (dy * xh).sum(0)
        dxh = dy * g
        dx = r * (dxh - xh * (dxh * xh).mean(-1, keepdims=True))
        return dx, dg
