"""Full-parameter PPO update (K11 / K12) against the fp64 oracle backward.

The reference's toy_rlhf_step updates every policy parameter by ascent on the
clipped surrogate (ppo.cpp:281-317, gradient ppo.cpp:138-177) and fits the
values toward discounted returns (ppo.cpp:292-315).  The engine does the same
through every layer of the actor and the critic (train_heads = 2): one update
on the engine, and the oracle's gradient (oracle/gpt_np.py, fp64, checked
against finite differences in tests/test_oracle_np.py) times the learning
rate must equal the change of EVERY trained tensor.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import gpt_np as N  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2509_25762_b200 import abi  # noqa: E402
from paper_2509_25762_b200.engine import Engine  # noqa: E402

pytestmark = pytest.mark.gpu

SAMPLE_SEED = 2
NAMES = ("embed", "final_norm", "head", "ln1", "wqkv", "bqkv", "wo", "ln2", "wgu", "wdown")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def snapshot(eng, model):
    dims, w = eng.export_weights(model)
    return dims, {k: (np.array(v, dtype=np.float64) if not isinstance(v, list) else
                      [np.array(x, dtype=np.float64) for x in v]) for k, v in w.items() if v is not None}


def oracle_update(eng, ids, P, hp, w_actor, w_critic, dims_a, dims_c):
    """Expected per-tensor deltas (lr * grad of the objective for the actor,
    -vlr * grad of the value loss for the critic) from the fp64 oracle."""
    ros = [eng.read_rollout(i) for i in ids]
    seqs = [np.concatenate([eng.read_prompt(i), ro["tokens"]]).astype(np.int64) for i, ro in zip(ids, ros)]
    # advantages exactly as the engine forms them: KL-shaped rewards, GAE, whitening
    adv_all, old_all, tok_all, ret_all = [], [], [], []
    for ro in ros:
        kl = ro["old_lp"].astype(np.float64) - ro["ref_lp"]
        r = -hp.kl_coef * kl
        r[-1] += ro["reward"]
        vals = np.concatenate([ro["values"], [0.0]])
        adv_all.append(np.array(O.gae(list(r), list(vals), hp.gamma, hp.lambda_)))
        old_all.append(ro["old_lp"].astype(np.float64))
        tok_all.append(ro["tokens"])
        L = ro["length"]
        ret_all.append(ro["reward"] * hp.gamma ** np.arange(L - 1, -1, -1.0))  # ppo.cpp:296-314
    adv = np.concatenate(adv_all)
    adv = (adv - adv.mean()) / np.sqrt(adv.var() + 1e-8)
    Ntok = len(adv)
    # actor
    actor = N.GptNp(dims_a, w_actor)
    caches, news, hfs = [], [], []
    for seq, ro in zip(seqs, ros):
        L = ro["length"]
        hf, lg, cache = actor.forward(seq[:-1], rows=np.arange(P - 1, P + L - 1), keep=True)
        lp = lg - lg.max(-1, keepdims=True)
        lp = lp - np.log(np.exp(lp).sum(-1, keepdims=True))
        news.append(lp[np.arange(L), ro["tokens"]])
        caches.append((cache, lg, hf))
    new = np.concatenate(news)
    obj, dobj = O.ppo_clip(list(new), list(np.concatenate(old_all)), list(adv), hp.clip_epsilon)
    dobj = np.asarray(dobj)
    ga = None
    k = 0
    for (cache, lg, hf), ro in zip(caches, ros):
        L = ro["length"]
        p = np.exp(lg - lg.max(-1, keepdims=True))
        p /= p.sum(-1, keepdims=True)
        G = -p * dobj[k:k + L, None]
        G[np.arange(L), ro["tokens"]] += dobj[k:k + L]
        k += L
        d_hf = np.zeros((hf.shape[0], hf.shape[1]))
        d_hf[P - 1:] = G @ actor.lm_head
        g = actor.backward(cache, d_hf)
        g["embed"] = g["embed"] + G.T @ hf[P - 1:]  # tied lm_head
        ga = g if ga is None else _add(ga, g)
    # critic
    critic = N.GptNp(dims_c, w_critic)
    ret = np.concatenate(ret_all)
    gc = None
    k = 0
    vloss = 0.0
    for seq, ro in zip(seqs, ros):
        L = ro["length"]
        hf, _, cache = critic.forward(seq[:-1], logits=False, keep=True)
        v = hf[P - 1:] @ critic.head
        e = v - ret[k:k + L]
        vloss += float((e * e).sum())
        dv = e / Ntok
        k += L
        d_hf = np.zeros_like(hf)
        d_hf[P - 1:] = np.outer(dv, critic.head)
        g = critic.backward(cache, d_hf)
        g["head"] = dv @ hf[P - 1:]
        gc = g if gc is None else _add(gc, g)
    da = _scale(ga, hp.learning_rate)
    dc = _scale(gc, -hp.value_learning_rate)
    return da, dc, obj, 0.5 * vloss / Ntok


def _add(a, b):
    return {k: ([x + y for x, y in zip(a[k], b[k])] if isinstance(a[k], list) else a[k] + b[k]) for k in a}


def _scale(a, s):
    return {k: ([x * s for x in v] if isinstance(v, list) else v * s) for k, v in a.items()}


def compare(delta_engine, delta_oracle, tol, who):
    worst = {}
    for k in NAMES:
        if k not in delta_oracle:
            continue
        eo, oo = delta_engine[k], delta_oracle[k]
        pairs = zip(eo, oo) if isinstance(oo, list) else [(eo, oo)]
        for li, (e, o) in enumerate(pairs):
            e = np.asarray(e).reshape(-1)
            o = np.asarray(o).reshape(-1)
            scale = max(np.abs(o).max(), 1e-12)
            err = np.abs(e - o).max() / scale
            worst[f"{k}[{li}]"] = err
            assert err <= tol, (who, k, li, err, scale)
            assert scale > 0, (who, k, li)
    return worst


def test_full_update_every_tensor_vs_oracle_fp32():
    P, C = 8, 16
    lens = [40, 64, 23, 64, 7]
    eng = Engine("tiny", dtype=abi.DTYPE_F32, max_slots=8, max_prompt_len=P, max_response_len=64,
                 sample_seed=SAMPLE_SEED, train_heads=2)
    st = [dict(id=i, prompt_len=P, target_len=L) for i, L in enumerate(lens)]
    eng.admit(st)
    eng.run_step(st, C, abi.MODE_STREAMED, len(lens))
    dims_a, wa0 = snapshot(eng, 0)
    dims_c, wc0 = snapshot(eng, 2)
    hp = abi.PpoHparams(gamma=1.0, lambda_=0.95, clip_epsilon=0.2, learning_rate=0.05,
                        value_learning_rate=0.02, kl_coef=0.05, whiten=1, value_target=abi.VALUE_MC_RETURN)
    ids = [s["id"] for s in st]
    da, dc, obj, vloss = oracle_update(eng, ids, P, hp, wa0, wc0, dims_a, dims_c)
    stats = eng.ppo_update(ids, hp)
    _, wa1 = snapshot(eng, 0)
    _, wc1 = snapshot(eng, 2)
    ea = {k: ([y - x for x, y in zip(wa0[k], wa1[k])] if isinstance(wa0[k], list) else wa1[k] - wa0[k]) for k in wa0}
    ec = {k: ([y - x for x, y in zip(wc0[k], wc1[k])] if isinstance(wc0[k], list) else wc1[k] - wc0[k]) for k in wc0}
    wa = compare(ea, da, 2e-3, "actor")
    wc = compare(ec, dc, 2e-3, "critic")
    print("actor", {k: f"{v:.1e}" for k, v in wa.items()})
    print("critic", {k: f"{v:.1e}" for k, v in wc.items()})
    assert abs(stats.ppo_objective - obj) < 1e-4
    assert abs(stats.value_loss - vloss) <= 1e-4 * max(1.0, vloss)
    eng.close()


W05 = dict(n_layers=2, d_model=896, n_heads=14, n_kv_heads=2, head_dim=64, d_ff=4864, vocab=151936, tied=1)
W15 = dict(n_layers=2, d_model=1536, n_heads=12, n_kv_heads=2, head_dim=128, d_ff=8960, vocab=151936, tied=1)


@pytest.mark.parametrize("shape", [W05, W15], ids=["0.5b-width", "1.5b-width"])
@pytest.mark.parametrize("simt", [0, 1], ids=["mma-attn", "simt-attn"])
def test_full_update_bf16_vs_oracle(shape, simt, monkeypatch):
    """bf16 engine (tcgen05 GEMMs, tensor-core or SIMT training attention,
    fp32 masters) at the 0.5B / 1.5B layer geometry (head_dim 64 / 128) and
    vocabulary (2 layers): every tensor's update agrees with the fp64 oracle
    gradient in direction (cosine >= 0.99) and size (max error <= 10% of the
    tensor's largest change; bf16 operands carry ~3 significant digits)."""
    if simt:
        monkeypatch.setenv("OPPO_TRAIN_SIMT_ATTN", "1")
    P, C = 16, 16
    lens = [40, 64, 23, 100]
    eng = Engine(shape, dtype=abi.DTYPE_BF16, max_slots=8, max_prompt_len=P, max_response_len=128,
                 sample_seed=SAMPLE_SEED, train_heads=2)
    st = [dict(id=i, prompt_len=P, target_len=L) for i, L in enumerate(lens)]
    eng.admit(st)
    eng.run_step(st, C, abi.MODE_STREAMED, len(lens))
    dims_a, wa0 = snapshot(eng, 0)
    dims_c, wc0 = snapshot(eng, 2)
    hp = abi.PpoHparams(gamma=1.0, lambda_=0.95, clip_epsilon=0.2, learning_rate=0.5,
                        value_learning_rate=0.05, kl_coef=0.05, whiten=1, value_target=abi.VALUE_MC_RETURN)
    ids = [s["id"] for s in st]
    da, dc, obj, vloss = oracle_update(eng, ids, P, hp, wa0, wc0, dims_a, dims_c)
    eng.ppo_update(ids, hp)
    # masters hold the un-rounded update: compare the fp32 masters' change
    ma1 = eng_masters(eng, 0)
    mc1 = eng_masters(eng, 2)
    for who, m1, w0, dd in (("actor", ma1, wa0, da), ("critic", mc1, wc0, dc)):
        for k in NAMES:
            if k not in dd:
                continue
            o_list = dd[k] if isinstance(dd[k], list) else [dd[k]]
            w_list = w0[k] if isinstance(w0[k], list) else [w0[k]]
            m_list = m1[k] if isinstance(m1[k], list) else [m1[k]]
            for li, (o, w, m) in enumerate(zip(o_list, w_list, m_list)):
                e = (np.asarray(m) - np.asarray(w)).reshape(-1)
                o = np.asarray(o).reshape(-1)
                cos = float(e @ o / (np.linalg.norm(e) * np.linalg.norm(o) + 1e-30))
                err = float(np.abs(e - o).max() / max(np.abs(o).max(), 1e-30))
                assert cos >= 0.99 and err <= 0.10, (who, k, li, cos, err)
    eng.close()


def eng_masters(eng, model):
    """fp32 masters (matrices) / fp32 parameters (vectors) after the update."""
    d, w = eng.export_weights(model, masters=True)
    return w
