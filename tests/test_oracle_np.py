"""The vectorised numpy oracle (oracle/gpt_np.py) against the scalar C oracle
(oracle_gpt_forward) and its backward against central finite differences."""
import numpy as np
import pytest

from oracle import gpt_np as N
from oracle import oracle as O

DIMS = dict(n_layers=2, d_model=64, n_heads=4, n_kv_heads=2, head_dim=16, d_ff=64, vocab=97, tied=0)


def rand_weights(d, seed=0, std=0.2):
    rng = np.random.default_rng(seed)
    D, H, KV, hd, F, V, L = (d["d_model"], d["n_heads"], d["n_kv_heads"], d["head_dim"], d["d_ff"],
                             d["vocab"], d["n_layers"])
    qkv = (H + 2 * KV) * hd
    f = lambda *s: (rng.standard_normal(s) * std).astype(np.float32)
    return {"embed": f(V, D), "lm_head": f(V, D), "final_norm": 1 + f(D),
            "ln1": [1 + f(D) for _ in range(L)], "wqkv": [f(qkv, D) for _ in range(L)],
            "bqkv": [f(qkv) for _ in range(L)], "wo": [f(D, H * hd) for _ in range(L)],
            "ln2": [1 + f(D) for _ in range(L)], "wgu": [f(2 * F, D) for _ in range(L)],
            "wdown": [f(D, F) for _ in range(L)], "head": f(D)}


def test_numpy_forward_matches_c_oracle():
    w = rand_weights(DIMS)
    tok = np.random.default_rng(1).integers(0, DIMS["vocab"], 23).astype(np.int32)
    h_c, lg_c = O.GptOracle(DIMS, w).forward(tok)
    h_n, lg_n = N.GptNp(DIMS, w).forward(tok)
    assert np.max(np.abs(h_c - h_n)) < 1e-10
    assert np.max(np.abs(lg_c - lg_n)) < 1e-10


def test_bf16_rounding():
    x = np.array([1.0, 1.00390625, 1.005859375, -3.14159, 1e-3])
    r = N.bf16(x)
    assert r[0] == 1.0 and r[1] == 1.0  # tie to even
    assert r[2] == 1.0078125
    assert abs(r[3] + 3.140625) < 1e-12


@pytest.mark.parametrize("target", ["logits", "head"])
def test_backward_matches_finite_differences(target):
    """Loss = sum(c * logits) (actor) or sum(c * hidden.head) (critic)."""
    w = rand_weights(DIMS, seed=3)
    tok = np.random.default_rng(4).integers(0, DIMS["vocab"], 11)
    m = N.GptNp(DIMS, w)
    rng = np.random.default_rng(5)
    c = rng.standard_normal((len(tok), DIMS["vocab"])) if target == "logits" else rng.standard_normal(len(tok))

    def loss(model):
        hf, lg = model.forward(tok)
        return float((c * lg).sum()) if target == "logits" else float((hf @ model.head * c).sum())

    hf, lg, cache = m.forward(tok, keep=True)
    d_hf = c @ m.lm_head if target == "logits" else np.outer(c, m.head)
    g = m.backward(cache, d_hf)
    for name, li, idx in [("wqkv", 0, (5, 7)), ("bqkv", 1, (3,)), ("wo", 1, (2, 9)), ("wgu", 0, (17, 4)),
                          ("wdown", 1, (8, 30)), ("ln1", 0, (6,)), ("ln2", 1, (11,)), ("final_norm", None, (13,)),
                          ("embed", None, (int(tok[2]), 5))]:
        arr = getattr(m, name) if li is None else m.layers[li][name]
        old = arr[idx]
        e = 1e-6
        arr[idx] = old + e
        lp = loss(m)
        arr[idx] = old - e
        lm = loss(m)
        arr[idx] = old
        fd = (lp - lm) / (2 * e)
        an = g[name][idx] if li is None else g[name][li][idx]
        assert abs(fd - an) <= 1e-6 * max(1.0, abs(fd)), (name, fd, an)


def _port_from(w, d):
    """The CPU port (oracle/cpu_step.py, the reference arm's workload) with the
    given weights instead of its timing constants."""
    from oracle import cpu_step as P
    port = P.Port(d)
    f = lambda a: np.asarray(a, dtype=np.float32)
    port.embed, port.lm_head, port.gf = f(w["embed"]), f(w["lm_head"]), f(w["final_norm"])
    for l, Lw in enumerate(port.layers):
        Lw.update(wqkv=f(w["wqkv"][l]), bqkv=f(w["bqkv"][l]), wo=f(w["wo"][l]), wgu=f(w["wgu"][l]),
                  wdown=f(w["wdown"][l]), g1=f(w["ln1"][l]), g2=f(w["ln2"][l]))
    return port


def test_cpu_port_computes_the_oracle_model():
    """The all-cores CPU port that bench.py times as the reference arm runs
    the same model as the fp64 oracle: prefill forward, one KV-cache decode
    step (logits of the last position) and the backward's weight gradients,
    within fp32 rounding."""
    w = rand_weights(DIMS, seed=7)
    d = DIMS
    tok = np.random.default_rng(8).integers(0, d["vocab"], 19)
    ref = N.GptNp(d, w)
    hf_r, lg_r, cache_r = ref.forward(tok, keep=True)
    port = _port_from(w, d)
    hf_p, cache_p = port.forward(tok, keep=True)
    assert np.abs(hf_p - hf_r).max() < 2e-4
    # decode the last token against the cache of the first T-1 positions
    T, KV, hd, G = len(tok), d["n_kv_heads"], d["head_dim"], d["n_heads"] // d["n_kv_heads"]
    _, (acts, *_rest) = port.forward(tok[:-1], keep=True)
    kv = []
    for a in acts:
        K = np.zeros((1, KV, T, hd), np.float32)
        V = np.zeros((1, KV, T, hd), np.float32)
        K[0, :, :T - 1] = a["kk"][::G]
        V[0, :, :T - 1] = a["vv"][::G]
        kv.append((K, V))
    lg_dec = port.decode_iteration(1, T, kv, np.random.default_rng(0), tok=[tok[-1]], return_logits=True)
    assert np.abs(lg_dec[0] - lg_r[-1]).max() < 5e-4 * max(1.0, np.abs(lg_r[-1]).max())
    # backward of sum(c * hidden) through every layer
    c = np.random.default_rng(9).standard_normal(hf_r.shape)
    g_r = ref.backward(cache_r, c)
    g_p = port.backward(cache_p, c.astype(np.float32))
    for l in range(d["n_layers"]):
        gp = g_p[d["n_layers"] - 1 - l]  # port returns layers last-first
        for name in ("wdown", "wgu", "wo", "wqkv", "bqkv"):
            a, b = gp[name], g_r[name][l]
            assert np.abs(a - b).max() <= 1e-3 * max(1.0, np.abs(b).max()), (l, name)
