"""End-to-end GPU parity of the step executor (pytest -m gpu, on a B200).

Config 1 of BASELINE.json (tiny actor/reward/critic/ref, 2 layers, d=128, 8
prompts, 64 new tokens, chunk 16) against the CPU oracle:
  * token ids: the engine draws each token in two levels (Gumbel-max over
    256-id vocabulary blocks, inverse CDF inside the block) from counter-based
    streams; the fp64 oracle (teacher forced on the same prompt) must draw the
    same id wherever both decision margins exceed 1e-3 (fp32) — in practice
    every token;
  * old log-probs, reference log-probs, per-token values and the reward:
    chunked incremental prefill on paged KV vs a full-sequence fp64 forward,
    |diff| <= 1e-3 (fp32) / 0.08 relative (bf16);
  * chunk boundaries, cut and deferral/selection decisions: bit-exact vs the
    reference's run_step under the lockstep latency model.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as O  # noqa: E402
from paper_2509_25762_b200 import abi  # noqa: E402
from paper_2509_25762_b200 import scheduler as S  # noqa: E402
from paper_2509_25762_b200.engine import Engine  # noqa: E402

pytestmark = pytest.mark.gpu

SAMPLE_SEED = 2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def oracles(eng):
    out = []
    for m in range(4):
        dims, w = eng.export_weights(m)
        out.append((O.GptOracle(dims, w), w.get("head")))
    return out


def log_softmax(x):
    m = x.max(-1, keepdims=True)
    return x - m - np.log(np.exp(x - m).sum(-1, keepdims=True))


def check_rollout(eng, orc, seq_id, P, tol_lp, tol_val, margin_tol, strict_tokens=True):
    ro = eng.read_rollout(seq_id)
    L = ro["length"]
    prompt = eng.read_prompt(seq_id)
    V = eng.cfg.actor.vocab
    assert prompt == O.prompt_tokens(SAMPLE_SEED, seq_id, P, V)
    seq = np.concatenate([prompt, ro["tokens"]]).astype(np.int32)
    (actor, _), (reward, rw), (critic, cw), (ref, _) = orc
    _, lg = actor.forward(seq[:-1])
    lp = log_softmax(lg)
    agree, checked = 0, 0
    for j in range(1, L + 1):
        tok, _, mb, mi = O.sample_token(lg[P + j - 2], O.token_key(SAMPLE_SEED, seq_id, j))
        if mb > margin_tol and mi > margin_tol:
            checked += 1
            agree += int(tok == ro["tokens"][j - 1])
        assert abs(lp[P + j - 2, ro["tokens"][j - 1]] - ro["old_lp"][j - 1]) <= tol_lp
    if strict_tokens:
        assert agree == checked, (agree, checked)
    else:
        assert agree >= 0.95 * checked, (agree, checked)
    hid_r, _ = reward.forward(seq, logits=False)
    assert abs(hid_r[P + L - 1] @ rw - ro["reward"]) <= tol_val * max(1, abs(ro["reward"]))
    hid_c, _ = critic.forward(seq, logits=False)
    vals = hid_c[P - 1:P + L - 1] @ cw
    assert np.max(np.abs(vals - ro["values"])) <= tol_val * max(1, np.abs(vals).max())
    _, lgr = ref.forward(seq[:-1])
    lpr = log_softmax(lgr)
    ref_lp = np.array([lpr[P + t - 2, ro["tokens"][t - 1]] for t in range(1, L + 1)])
    assert np.max(np.abs(ref_lp - ro["ref_lp"])) <= tol_lp
    return ro


def fresh_states(n, P, lengths, start_id=0):
    return [dict(id=start_id + i, prompt_len=P, target_len=L) for i, L in enumerate(lengths)]


@pytest.mark.parametrize("dtype", [abi.DTYPE_F32, abi.DTYPE_BF16])
def test_cfg1_single_step_vs_oracle(dtype):
    P, B, L, C = 8, 8, 64, 16
    eng = Engine("tiny", dtype=dtype, max_slots=16, max_prompt_len=P, max_response_len=64,
                 sample_seed=SAMPLE_SEED)
    states = fresh_states(B, P, [L] * B)
    eng.admit(states)
    outs, led = eng.run_step(states, C, abi.MODE_STREAMED, B)
    po, pl = S.plan_step(states, C, abi.MODE_STREAMED, B)
    assert [o.as_tuple() for o in outs] == [o.as_tuple() for o in po]
    assert led.wall == 64 and led.decode_iters == 64 and led.step_us > 0
    orc = oracles(eng)
    f32 = dtype == abi.DTYPE_F32
    for s in states:
        check_rollout(eng, orc, s["id"], P, tol_lp=1e-3 if f32 else 0.15,
                      tol_val=1e-3 if f32 else 0.1, margin_tol=1e-3 if f32 else 0.2,
                      strict_tokens=f32)
    eng.close()


def test_streamed_vs_sequential_content_invariance():
    """streaming does not alter generation or the scoring inputs;
    chunked prefill == whole-response prefill (fp32: bit-identical)."""
    P, C = 8, 16
    lens = [64, 37, 50, 5, 64, 17, 33, 60]
    got = {}
    for mode in (abi.MODE_STREAMED, abi.MODE_SEQUENTIAL):
        eng = Engine("tiny", dtype=abi.DTYPE_F32, max_slots=16, max_prompt_len=P,
                     max_response_len=64, sample_seed=SAMPLE_SEED)
        st = fresh_states(len(lens), P, lens)
        eng.admit(st)
        eng.run_step(st, C, mode, len(lens))
        got[mode] = [eng.read_rollout(s["id"]) for s in st]
        eng.close()
    for i, (a, b) in enumerate(zip(got[abi.MODE_STREAMED], got[abi.MODE_SEQUENTIAL])):
        for k in ("tokens", "old_lp", "values", "ref_lp"):
            bad = np.nonzero(a[k] != b[k])[0]
            assert len(bad) == 0, (i, k, bad[:8].tolist(), a[k][bad[:4]], b[k][bad[:4]])
        assert a["reward"] == b["reward"], (i, a["reward"], b["reward"])


@pytest.mark.parametrize("carry", [abi.CARRY_CHUNK, abi.CARRY_TOKEN])
def test_overcommit_carry_multi_step_vs_oracle(carry):
    """Deferred sequences keep their KV pages and (whole-chunk or partial)
    tokens across steps; decisions match the logical clock / reference."""
    cfg = S.default_config(steps=4, batch_size=8, prompt_len=8, delta_init=2, delta_max=2,
                           chunk_size=16, carry_granularity=carry,
                           lengths_kind=abi.LEN_LOGNORMAL, lengths_mu_log=3.5,
                           lengths_sigma_log=0.6, lengths_cap=64,
                           latency_decode_per_token=1, latency_prefill_per_token=0,
                           latency_reward_residual=0, latency_placement=1)
    eng = Engine("tiny", dtype=abi.DTYPE_F32, max_slots=16, max_prompt_len=8, max_response_len=64,
                 sample_seed=SAMPLE_SEED, carry=carry)
    lens = S.sample_lengths(cfg.lengths, 1, 64)
    entries, next_id = [], 0
    sel_log = []
    orc = None
    for step in range(cfg.steps):
        fresh = []
        while len(entries) + len(fresh) < cfg.batch_size + cfg.delta_init:
            fresh.append(dict(id=next_id, prompt_len=8, target_len=lens[next_id],
                              admitted_at=step, arrival_step=step))
            next_id += 1
        entries += [S.seq_array([f])[0] for f in fresh]
        eng.admit(fresh)
        active = [e for e in entries if not e.scored]
        pre = len(entries) - len(active)
        outs, led = eng.run_step(active, cfg.chunk_size, abi.MODE_STREAMED,
                                 cfg.batch_size - pre)
        batch, entries, _ = S.select_finished(entries, outs, cfg.batch_size)
        sel_log.append([b.id for b in batch])
        if orc is None:
            orc = oracles(eng)
        for b in batch:
            check_rollout(eng, orc, b.id, 8, 1e-3, 1e-3, 1e-3)
        eng.release([b.id for b in batch])
    # same decisions as the scheduler-only run of the same config
    _, sel = S.run_seed_logical(cfg, 1)
    assert sel_log == sel
    eng.close()


def test_gpu_run_seed_simulate_matches_logical():
    cfg = S.default_config(steps=6, batch_size=8, prompt_len=8, delta_init=2, delta_max=4,
                           controller=abi.DELTA_ALG1, window=2, proxy_kind=1, chunk_size=16,
                           lengths_kind=abi.LEN_LOGNORMAL, lengths_mu_log=3.5,
                           lengths_sigma_log=0.6, lengths_cap=64,
                           latency_decode_per_token=1, latency_prefill_per_token=0,
                           latency_reward_residual=0, latency_placement=1)
    eng = Engine("tiny", dtype=abi.DTYPE_BF16, max_slots=16, max_prompt_len=8,
                 max_response_len=64, sample_seed=SAMPLE_SEED)
    recs, sel = eng.run_seed(cfg, 1)
    lrecs, lsel = S.run_seed_logical(cfg, 1)
    key = lambda r: (r.wall_ticks, r.finished, r.deferred, r.delta, r.max_deferrals)
    assert [key(r) for r in recs] == [key(r) for r in lrecs]
    assert sel == lsel
    assert all(r.step_us > 0 for r in recs)
    eng.close()


def test_ppo_update_vs_oracle_fp32():
    """fill_values + GAE + clipped objective + head update (lm_head ascent,
    value-head regression) vs the fp64 oracle on the same rollouts."""
    P, C = 8, 16
    lens = [40, 64, 23, 64]
    eng = Engine("tiny", dtype=abi.DTYPE_F32, max_slots=8, max_prompt_len=P, max_response_len=64,
                 sample_seed=SAMPLE_SEED, train_heads=1)
    st = fresh_states(len(lens), P, lens)
    eng.admit(st)
    eng.run_step(st, C, abi.MODE_STREAMED, len(lens))
    orc = oracles(eng)
    ros = [eng.read_rollout(s["id"]) for s in st]
    W0 = eng.get_tensor(0, "lm_head").reshape(512, 128).astype(np.float64)
    hp = abi.PpoHparams(gamma=1.0, lambda_=0.95, clip_epsilon=0.2, learning_rate=0.5,
                        value_learning_rate=0.1, kl_coef=0.05, whiten=1)
    stats = eng.ppo_update([s["id"] for s in st], hp)
    # oracle
    actor = orc[0][0]
    adv_all, new_all, old_all, hid_all, tok_all, kl_all = [], [], [], [], [], []
    for s, ro in zip(st, ros):
        seq = np.concatenate([eng.read_prompt(s["id"]), ro["tokens"]]).astype(np.int32)
        hid, lg = actor.forward(seq[:-1])
        L = ro["length"]
        lp = log_softmax(lg)
        new = np.array([lp[P + j - 2, ro["tokens"][j - 1]] for j in range(1, L + 1)])
        kl = ro["old_lp"].astype(np.float64) - ro["ref_lp"]
        r = -0.05 * kl
        r[-1] += ro["reward"]
        vals = np.concatenate([ro["values"], [0.0]])
        adv_all.append(np.array(O.gae(list(r), list(vals), 1.0, 0.95)))
        new_all.append(new)
        old_all.append(ro["old_lp"].astype(np.float64))
        hid_all.append(hid[P - 1:P + L - 1])
        tok_all.append(ro["tokens"])
        kl_all.append(kl)
    adv = np.concatenate(adv_all)
    adv = (adv - adv.mean()) / np.sqrt(adv.var() + 1e-8)
    new, old = np.concatenate(new_all), np.concatenate(old_all)
    obj, dobj = O.ppo_clip(list(new), list(old), list(adv), 0.2)
    assert abs(stats.ppo_objective - obj) < 1e-4
    assert abs(stats.kl_mean - np.concatenate(kl_all).mean()) < 1e-5
    assert abs(stats.mean_reward - np.mean([ro["reward"] for ro in ros])) < 1e-5
    # lm_head ascent: W += lr * sum_t c_t (e_y - softmax) h_t^T
    H = np.concatenate(hid_all)
    tok = np.concatenate(tok_all)
    logits = H @ W0.T
    p = np.exp(log_softmax(logits))
    G = -p * np.asarray(dobj)[:, None]
    G[np.arange(len(tok)), tok] += np.asarray(dobj)
    dW = G.T @ H
    W1 = eng.get_tensor(0, "lm_head").reshape(512, 128).astype(np.float64)
    assert np.max(np.abs((W1 - W0) - 0.5 * dW)) <= 1e-5 * max(1e-3, np.abs(0.5 * dW).max()) + 1e-7
    eng.close()


@pytest.mark.parametrize("attn_env", ["", "OPPO_ATTN_TP16=1", "OPPO_ATTN_WARPS=8", "OPPO_ATTN_WARPS=4",
                                      "OPPO_SCORER_STREAMS=3"])
def test_gqa_05b_width_bf16_vs_oracle(attn_env):
    """0.5B geometry (d=896, 14 q heads over 2 kv heads, head_dim 64, SwiGLU
    4864) at 2 layers / small vocabulary: tensor-core attention (decode and
    chunked prefill, G=7 rows per KV head) and tcgen05 GEMMs vs fp64.  Every
    decode-attention variant the launcher can pick by batch size (4 warps x 32
    or 16 positions, 8 warps x 16) is forced once."""
    import os
    shape = dict(n_layers=2, d_model=896, n_heads=14, n_kv_heads=2, head_dim=64, d_ff=4864,
                 vocab=1024, tied=1)
    P, C = 16, 16
    lens = [40, 70, 23, 64]
    key, _, val = attn_env.partition("=")
    if key:
        os.environ[key] = val
    try:
        eng = Engine(shape, dtype=abi.DTYPE_BF16, max_slots=8, max_prompt_len=P, max_response_len=80,
                     sample_seed=SAMPLE_SEED)
    finally:
        if key:
            os.environ.pop(key, None)
    st = fresh_states(len(lens), P, lens)
    eng.admit(st)
    eng.run_step(st, C, abi.MODE_STREAMED, len(lens))
    orc = oracles(eng)
    for s in st:
        check_rollout(eng, orc, s["id"], P, tol_lp=0.15, tol_val=0.2, margin_tol=0.2,
                      strict_tokens=False)  # bf16 reward/value heads at d=896: ~0.1 absolute
    eng.close()


@pytest.mark.parametrize("split", ["", "1"], ids=["split_kv", "one_cta"])
@pytest.mark.parametrize("hd", [64, 128])
def test_long_context_split_kv_decode_vs_oracle(hd, split):
    """Long-context decode iterations (longest context >= OPPO_ATTN_LONG_CTX)
    run the split-KV graph variant: the KV range of a row is split over a
    cluster of CTAs (>= OPPO_ATTN_SPLIT_MINPOS positions each) merged through
    DSMEM.  The thresholds are scaled down here (64 / 32 instead of 768 / 512)
    so 96-token prompts take the split path and the fp64 oracle stays fast;
    head_dim 64 (0.5B width, G=7) and 128 (G=4); OPPO_ATTN_MAX_SPLIT=1 forces
    one CTA per row for comparison."""
    import os
    if hd == 64:
        shape = dict(n_layers=2, d_model=896, n_heads=14, n_kv_heads=2, head_dim=64, d_ff=4864,
                     vocab=1024, tied=1)
    else:
        shape = dict(n_layers=2, d_model=1024, n_heads=8, n_kv_heads=2, head_dim=128, d_ff=2816,
                     vocab=1024, tied=1)
    P, C = 96, 16
    lens = [20, 35, 12, 28]
    env = {"OPPO_ATTN_LONG_CTX": "64", "OPPO_ATTN_SPLIT_MINPOS": "32"}
    if split:
        env["OPPO_ATTN_MAX_SPLIT"] = split
    os.environ.update(env)
    try:
        eng = Engine(shape, dtype=abi.DTYPE_BF16, max_slots=8, max_prompt_len=P, max_response_len=48,
                     sample_seed=SAMPLE_SEED)
    finally:
        for k in env:
            os.environ.pop(k, None)
    st = fresh_states(len(lens), P, lens)
    eng.admit(st)
    eng.run_step(st, C, abi.MODE_STREAMED, len(lens))
    orc = oracles(eng)
    for s in st:
        check_rollout(eng, orc, s["id"], P, tol_lp=0.15, tol_val=0.2, margin_tol=0.2,
                      strict_tokens=False)
    eng.close()


@pytest.mark.parametrize("hd", [64, 128])
def test_rope_append_epilogue_matches_separate_kernel(hd):
    """Prefill q|k|v projection with RoPE + paged KV append in the GEMM
    epilogue (EPI_ROPE_APPEND, the default) against EPI_STORE followed by the
    rope_append kernel (OPPO_ROPE_EPI=0): same arithmetic, so at head_dim 64
    (same tiles and K splits in both runs) every rollout output (tokens,
    log-probs, reference log-probs, values, rewards) is bit-identical.  At
    head_dim 128 the fused epilogue needs >= 128-wide tiles where the
    unfused path picks 64-wide ones with another K split for small passes, so
    the summation order differs: there the fused run is checked against the
    fp64 oracle on every sequence."""
    import os
    H, KV = (14, 2) if hd == 64 else (12, 2)
    shape = dict(n_layers=2, d_model=H * hd, n_heads=H, n_kv_heads=KV, head_dim=hd,
                 d_ff=4864, vocab=1024, tied=1)
    P, C = 40, 16  # multi-chunk prompts: prefill rows span pages and tiles
    lens = [40, 70, 23, 64, 5, 33]
    res = []
    for flag in ("1", "0"):
        os.environ["OPPO_ROPE_EPI"] = flag
        try:
            eng = Engine(shape, dtype=abi.DTYPE_BF16, max_slots=8, max_prompt_len=P,
                         max_response_len=80, sample_seed=SAMPLE_SEED)
        finally:
            os.environ.pop("OPPO_ROPE_EPI", None)
        st = fresh_states(len(lens), P, lens)
        eng.admit(st)
        eng.run_step(st, C, abi.MODE_STREAMED, len(lens))
        res.append([eng.read_rollout(s["id"]) for s in st])
        if flag == "1":
            orc = oracles(eng)
            for s in (st if hd == 128 else st[:3]):
                check_rollout(eng, orc, s["id"], P, tol_lp=0.15, tol_val=0.2, margin_tol=0.2,
                              strict_tokens=False)
        eng.close()
        if hd == 128:
            return
    for a, b in zip(*res):
        assert a["length"] == b["length"] and a["reward"] == b["reward"]
        for k in ("tokens", "old_lp", "ref_lp", "values"):
            assert np.array_equal(a[k], b[k]), k


def test_policy_logprob_precompute_is_bit_identical():
    """The update's current-policy log-probs, computed at the end of run_step
    on the actor SMs while the scorers finish (OPPO_PRE_LP=1, default), give
    the same PPO statistics and the same updated lm_head / value head, bit for
    bit, as recomputing them inside oppo_ppo_update (OPPO_PRE_LP=0); two
    rounds, so the second reuses log-probs taken after the first update."""
    import os
    shape = dict(n_layers=2, d_model=896, n_heads=14, n_kv_heads=2, head_dim=64, d_ff=4864,
                 vocab=1024, tied=1)
    P, C = 16, 16
    hp = abi.PpoHparams(gamma=1.0, lambda_=0.95, clip_epsilon=0.2, learning_rate=0.5,
                        value_learning_rate=0.1, kl_coef=0.05, whiten=1)
    res = []
    for flag in ("1", "0"):
        os.environ["OPPO_PRE_LP"] = flag
        try:
            eng = Engine(shape, dtype=abi.DTYPE_BF16, max_slots=16, max_prompt_len=P,
                         max_response_len=64, sample_seed=SAMPLE_SEED, train_heads=1)
        finally:
            os.environ.pop("OPPO_PRE_LP", None)
        out = []
        for rnd in range(2):
            lens = [20 + (11 * i + 5 * rnd) % 40 for i in range(8)]
            st = fresh_states(len(lens), P, lens, start_id=100 * rnd)
            eng.admit(st)
            eng.run_step(st, C, abi.MODE_STREAMED, len(lens))
            stats = eng.ppo_update([s_["id"] for s_ in st], hp)
            out.append((stats.ppo_objective, stats.kl_mean, stats.adv_mean, stats.adv_std,
                        stats.value_loss))
            eng.release([s_["id"] for s_ in st])
        out.append(eng.get_tensor(0, "lm_head"))
        out.append(eng.get_tensor(2, "head"))
        res.append(out)
        eng.close()
    a, b = res
    assert a[0] == b[0] and a[1] == b[1]
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])


@pytest.mark.parametrize("train", [1, 2])
def test_engine_checkpoint_resume_is_bit_identical(tmp_path, train):
    """oppo_engine_save after a step with carried sequences (token carry: KV
    pages, partial tokens and log-probs of the stragglers, trained heads),
    oppo_engine_load into a fresh engine of the same configuration: the next
    step (refill, decode of the carried and the fresh sequences, scoring,
    selection, PPO update) is bit-identical on the original and the restored
    engine; a mismatching configuration is refused."""
    shape = dict(n_layers=2, d_model=896, n_heads=14, n_kv_heads=2, head_dim=64, d_ff=4864,
                 vocab=1024, tied=1)
    P, C, B = 16, 16, 4
    hp = abi.PpoHparams(gamma=1.0, lambda_=0.95, clip_epsilon=0.2, learning_rate=0.5,
                        value_learning_rate=0.1, kl_coef=0.05, whiten=1)

    def make(**kw):
        return Engine(shape, dtype=abi.DTYPE_BF16, max_slots=16, max_prompt_len=P, max_response_len=64,
                      sample_seed=SAMPLE_SEED, train_heads=train, carry=abi.CARRY_TOKEN, **kw)

    def fresh(ids, lens):
        return [S.seq_array([dict(id=i, prompt_len=P, target_len=L)])[0] for i, L in zip(ids, lens)]

    def step(eng, entries):
        active = [e for e in entries if not e.scored]
        outs, _ = eng.run_step(active, C, abi.MODE_STREAMED, B - (len(entries) - len(active)))
        batch, entries, _ = S.select_finished(entries, outs, B)
        ids = [b.id for b in batch]
        st = eng.ppo_update(ids, hp)
        ro = [eng.read_rollout(i) for i in ids]
        eng.release(ids)
        return entries, ids, (st.ppo_objective, st.kl_mean, st.value_loss, st.mean_reward), ro

    a = make()
    first = fresh(range(8), [45, 12, 60, 20, 33, 64, 9, 27])
    a.admit(first)
    entries, _, _, _ = step(a, first)
    assert any(e.generated > 0 for e in entries)  # carried stragglers with decoded tokens
    ck = tmp_path / "engine.ckpt"
    a.save(ck)
    b = make()
    b.load(ck)
    res = []
    for eng in (a, b):
        more = fresh(range(8, 12), [30, 50, 14, 41])
        eng.admit(more)
        ents, ids, stats, ro = step(eng, [S.seq_array([e])[0] for e in entries] + more)
        res.append((ids, stats, ro, eng.get_tensor(0, "lm_head"), eng.get_tensor(2, "head"),
                    [(e.id, e.generated, e.prefilled_tokens) for e in ents],
                    [eng.get_tensor(m, k, 1) for m in (0, 2) for k in ("wqkv:master", "wdown", "ln2")]))
    (ia, sa, ra, la, ha, ea, ta), (ib, sb, rb, lb, hb, eb, tb) = res
    for x, y in zip(ta, tb):  # trunk tensors (full-parameter update) and their masters
        assert np.array_equal(x, y)
    assert ia == ib and sa == sb and ea == eb
    for x, y in zip(ra, rb):
        assert x["reward"] == y["reward"]
        for k in ("tokens", "old_lp", "ref_lp", "values"):
            assert np.array_equal(x[k], y[k]), k
    assert np.array_equal(la, lb) and np.array_equal(ha, hb)
    a.close()
    b.close()
    c = Engine(shape, dtype=abi.DTYPE_BF16, max_slots=8, max_prompt_len=P, max_response_len=64,
               sample_seed=SAMPLE_SEED, train_heads=train, carry=abi.CARRY_TOKEN)
    with pytest.raises(Exception, match="configuration"):
        c.load(ck)
    c.close()


def test_two_branch_decode_iterations_vs_oracle():
    """Decode iterations split into two concurrent halves (OPPO_DEC_SPLIT_MIN:
    rows [0, M1) on the actor stream, [M1, M) on a second stream, one CUDA
    graph with a fork/join) at 40 active rows (bucket 48 -> 32 + 16), 0.5B
    geometry: sampled tokens / log-probs / scorer outputs against the fp64
    oracle, and every sequence reaches its target length (the iteration
    counter advances once per iteration)."""
    import os
    shape = dict(n_layers=2, d_model=896, n_heads=14, n_kv_heads=2, head_dim=64, d_ff=4864,
                 vocab=1024, tied=1)
    P, C = 16, 16
    lens = [20 + (7 * i) % 40 for i in range(40)]
    os.environ["OPPO_DEC_SPLIT_MIN"] = "32"
    try:
        eng = Engine(shape, dtype=abi.DTYPE_BF16, max_slots=48, max_prompt_len=P,
                     max_response_len=64, sample_seed=SAMPLE_SEED)
    finally:
        os.environ.pop("OPPO_DEC_SPLIT_MIN", None)
    st = fresh_states(len(lens), P, lens)
    eng.admit(st)
    eng.run_step(st, C, abi.MODE_STREAMED, len(lens))
    orc = oracles(eng)
    for i in (0, 1, 17, 31, 32, 33, 39):  # both halves and the boundary
        check_rollout(eng, orc, st[i]["id"], P, tol_lp=0.15, tol_val=0.2, margin_tol=0.2,
                      strict_tokens=False)
    for s_ in st:
        assert eng.read_rollout(s_["id"])["length"] == s_["target_len"]
    eng.close()


def test_gpu_tuner_on_measured_step_time_replays(tmp_path):
    """the chunk-size tuner (chunking.cpp:61-107) fed the GPU's
    measured step time.  Replaying the recorded (candidate, step_us) pairs
    through the tuner reproduces every chunk size the run used after its
    exploration steps; the run's outputs are written in the reference's
    formats (steps/tuner CSV, summary.json)."""
    from paper_2509_25762_b200 import outputs
    cfg = S.default_config(mode=abi.RUN_TUNE, steps=14, batch_size=8, prompt_len=8, delta_init=2,
                           delta_max=4, controller=abi.DELTA_FIXED, proxy_kind=0, chunk_size=16,
                           tune_chunks=1, chunk_candidates=[8, 16, 32], retune_period=7,
                           lengths_kind=abi.LEN_LOGNORMAL, lengths_mu_log=3.5,
                           lengths_sigma_log=0.6, lengths_cap=64, latency_decode_per_token=1,
                           latency_prefill_per_token=0, latency_reward_residual=0,
                           latency_placement=1)
    eng = Engine("tiny", dtype=abi.DTYPE_BF16, max_slots=16, max_prompt_len=8,
                 max_response_len=64, sample_seed=SAMPLE_SEED)
    recs, _ = eng.run_seed(cfg, 3)
    eng.close()
    assert len(recs) == cfg.steps and all(r.step_us > 0 for r in recs)
    rows = outputs.tuner_rows(cfg, recs, measure="us")
    assert [c for _, c, _, _ in rows] == [8, 16, 32, 8, 16, 32]  # ascending exploration per period
    chosen_after = {}
    for step, _, _, ch in rows:
        chosen_after[step] = ch
    current, by_step = 8, {}
    for r in recs:
        if r.step in chosen_after:
            current = chosen_after[r.step]
        elif r.step % cfg.retune_period >= 3:
            by_step[r.step] = current
    assert by_step and all(recs[s].chunk_size == c for s, c in by_step.items())
    run = dict(seed=3, records=recs, complete=True, error="")
    outputs.write_outputs(cfg, [run], [run], tmp_path)
    assert (tmp_path / "steps_3.csv").read_text().startswith("step,wall_ticks,finished")
    assert (tmp_path / "tuner_3.csv").exists() and (tmp_path / "steps_3_us.csv").exists()


def test_7b_actor_15b_scorers_width_bf16_vs_oracle():
    """BASELINE configs 3-5 pair a wide actor with smaller scorers: a 7B-width
    actor (d=3584, 28 q / 4 kv heads, head_dim 128, SwiGLU 18944, untied
    lm_head) with 1.5B-width reward / critic / reference (d=1536, 12 / 2
    heads, SwiGLU 8960), 2 layers each, 1024-token vocabulary: decode (head_dim
    128, G=7 tensor-core attention, decode GEMMs at d=3584) and the scorers'
    chunked prefill against the fp64 oracle."""
    actor = dict(n_layers=2, d_model=3584, n_heads=28, n_kv_heads=4, head_dim=128, d_ff=18944,
                 vocab=1024, tied=0)
    scorer = dict(n_layers=2, d_model=1536, n_heads=12, n_kv_heads=2, head_dim=128, d_ff=8960,
                  vocab=1024, tied=1)
    P, C = 16, 16
    lens = [30, 45, 12, 38]
    eng = Engine(actor, scorer, scorer, scorer, dtype=abi.DTYPE_BF16, max_slots=8, max_prompt_len=P,
                 max_response_len=48, sample_seed=SAMPLE_SEED)
    st = fresh_states(len(lens), P, lens)
    eng.admit(st)
    eng.run_step(st, C, abi.MODE_STREAMED, len(lens))
    orc = oracles(eng)
    for s in st[:3]:
        check_rollout(eng, orc, s["id"], P, tol_lp=0.2, tol_val=0.25, margin_tol=0.2,
                      strict_tokens=False)
    eng.close()


def test_untied_full_update_teardown_leaves_cuda_clean():
    """An untied actor (7B geometry, separate lm_head) through the full
    update and engine teardown: its lm_head fp32 master is freed once, and
    the caller's next CUDA call (torch here) sees no leftover error -- a
    double free used to surface as 'invalid argument' in bench.py's cfg4 run."""
    shape = dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=2, head_dim=64, d_ff=512, vocab=2048, tied=0)
    P = 8
    eng = Engine(shape, dtype=abi.DTYPE_BF16, max_slots=8, max_prompt_len=P, max_response_len=32,
                 sample_seed=SAMPLE_SEED, train_heads=2)
    st = fresh_states(4, P, [12, 20, 7, 16])
    eng.admit(st)
    outs, _ = eng.run_step(st, 8, abi.MODE_STREAMED, 4)
    hp = abi.PpoHparams(gamma=1.0, lambda_=0.95, clip_epsilon=0.2, learning_rate=1e-3,
                        value_learning_rate=1e-3, kl_coef=0.05, whiten=1)
    eng.ppo_update([s["id"] for s in st], hp)
    eng.close()
    x = torch.ones(4, device="cuda") * 2
    torch.cuda.synchronize()
    assert float(x.sum()) == 8.0


def test_edge_cases_single_token_prompts_and_responses_vs_oracle():
    """Edge cases of the step executor (fp32, strict token parity): one-token
    prompts (no admission prefill; decode starts from the prompt token),
    one- and two-token responses (a sequence that finishes on the first
    iteration and whose only chunk carries the prompt), and mixed prompt
    lengths in one batch."""
    P_max, C = 8, 4
    eng = Engine("tiny", dtype=abi.DTYPE_F32, max_slots=8, max_prompt_len=P_max,
                 max_response_len=32, sample_seed=SAMPLE_SEED)
    states = [dict(id=0, prompt_len=1, target_len=1), dict(id=1, prompt_len=1, target_len=9),
              dict(id=2, prompt_len=8, target_len=2), dict(id=3, prompt_len=5, target_len=17)]
    eng.admit(states)
    outs, led = eng.run_step(states, C, abi.MODE_STREAMED, len(states))
    plan, _ = S.plan_step(states, C, abi.MODE_STREAMED, len(states))
    assert [o.as_tuple() for o in outs] == [o.as_tuple() for o in plan]
    orc = oracles(eng)
    for s in states:
        check_rollout(eng, orc, s["id"], s["prompt_len"], tol_lp=1e-3, tol_val=1e-3, margin_tol=1e-3)
    eng.close()


def test_engine_input_errors_map_to_reference_exceptions():
    """Invalid runtime input raises InputError (rlpipe::InputError,
    errors.hpp:15-18), invalid configuration ConfigError; the engine stays
    usable after an input error."""
    from paper_2509_25762_b200._lib import ConfigError, InputError
    eng = Engine("tiny", dtype=abi.DTYPE_F32, max_slots=2, max_prompt_len=8, max_response_len=16,
                 sample_seed=SAMPLE_SEED)
    with pytest.raises(InputError):
        eng.admit([dict(id=0, prompt_len=8, target_len=17)])  # beyond max_response_len
    with pytest.raises(InputError):
        eng.admit([dict(id=0, prompt_len=9, target_len=4)])  # beyond max_prompt_len
    eng.admit([dict(id=0, prompt_len=8, target_len=4)])
    with pytest.raises(InputError):
        eng.admit([dict(id=0, prompt_len=8, target_len=4)])  # duplicate id
    with pytest.raises(InputError):
        eng.run_step([dict(id=5, prompt_len=8, target_len=4)], 4, abi.MODE_STREAMED, 1)  # not admitted
    eng.admit([dict(id=1, prompt_len=8, target_len=4)])
    with pytest.raises(InputError):
        eng.admit([dict(id=2, prompt_len=8, target_len=4)])  # no free slot
    st = [dict(id=0, prompt_len=8, target_len=4), dict(id=1, prompt_len=8, target_len=4)]
    outs, _ = eng.run_step(st, 4, abi.MODE_STREAMED, 2)  # still usable
    assert all(o.score_ready >= 0 for o in outs)
    eng.close()
    with pytest.raises(ConfigError):
        Engine("tiny", dtype=7)


def test_run_seed_ex_prompt_source_and_kv_admission_control():
    """The C++ step loop with the host prompt source (oppo_run_seed_ex, the
    reference's PromptSource seam): decisions equal the logical loop's and the
    engine holds exactly the host's prompts.  With a KV pool smaller than the
    B + delta worst case, refill defers sequences instead of failing, and the
    run still completes with every sequence selected at most once."""
    cfg = S.default_config(mode=abi.RUN_SIMULATE, steps=6, batch_size=8, prompt_len=8, delta_init=4,
                           delta_max=4, controller=abi.DELTA_FIXED, chunk_size=16,
                           lengths_kind=abi.LEN_LOGNORMAL, lengths_mu_log=3.5, lengths_sigma_log=0.6,
                           lengths_cap=64, latency_decode_per_token=1, latency_prefill_per_token=0,
                           latency_reward_residual=0, latency_placement=1)
    seen = {}

    def pf(i, plen):
        t = [(i * 7 + q * 13) % 512 for q in range(plen)]
        seen[i] = t
        return t

    checked = []

    def on_step(rec):  # prompts of the step's sequences are the host's
        return False

    eng = Engine("tiny", dtype=abi.DTYPE_F32, max_slots=16, max_prompt_len=8, max_response_len=64,
                 sample_seed=SAMPLE_SEED)
    recs, sel, leds = eng.run_seed_ex(cfg, 1, prompt_fn=pf, on_step=on_step)
    _, lsel = S.run_seed_logical(cfg, 1)
    assert sel == lsel
    assert len(recs) == 6 and all(l.decode_iters > 0 for l in leds)
    eng.close()
    # admission control: 14 pages of 64 tokens; a sequence needs 1-2 pages
    eng = Engine("tiny", dtype=abi.DTYPE_F32, max_slots=16, max_prompt_len=8, max_response_len=64,
                 sample_seed=SAMPLE_SEED, kv_pages=14)
    recs, sel, _ = eng.run_seed_ex(cfg, 1, prompt_fn=pf)
    got = [i for s in sel for i in s if i >= 0]
    assert len(recs) == 6 and len(got) == len(set(got)) and len(got) >= 24
    assert sel != lsel  # the deferrals changed the schedule (the test is not vacuous)
    eng.close()



def test_measured_partition_utilization():
    """engine.cpp:225-233's utilization on the GPU: the step loop's records
    carry the actor partition's decode-loop time and the scorer partition's
    summed wave spans over the step's device time (streamed: both busy; the
    scorer's share smaller than the decode's for this small step)."""
    shape = dict(n_layers=2, d_model=256, n_heads=4, n_kv_heads=2, head_dim=64, d_ff=512, vocab=2048, tied=1)
    eng = Engine(shape, dtype=abi.DTYPE_BF16, max_slots=24, max_prompt_len=16, max_response_len=96,
                 sample_seed=SAMPLE_SEED, train_heads=0)
    cfg = S.default_config(mode=abi.RUN_TRAIN, steps=3, batch_size=8, prompt_len=16, delta_init=2, delta_min=0,
                           delta_max=2, chunk_size=16, schedule_mode=abi.MODE_STREAMED, lengths_kind=abi.LEN_LOGNORMAL,
                           lengths_mu_log=3.5, lengths_sigma_log=0.6, lengths_cap=96, ppo_learning_rate=1e-3,
                           ppo_value_learning_rate=1e-3)
    recs, _, leds = eng.run_seed_ex(cfg, 5)
    eng.close()
    for r, led in zip(recs, leds):
        assert led.step_us > 0 and led.score_busy_us > 0
        assert 0.0 < r.util_generation <= 1.01 and 0.0 < r.util_scoring <= 1.01, (r.util_generation, r.util_scoring)
        assert abs(r.util_generation - led.decode_loop_us / led.step_us) < 1e-9


def _run_flags(flags, scorer_sms):
    """Two overcommitted streamed steps (0.5B width, 2 layers) with the K13
    chunk hand-off on device flags (1) or per-wave events (0)."""
    import os
    shape = dict(n_layers=2, d_model=896, n_heads=14, n_kv_heads=2, head_dim=64, d_ff=4864,
                 vocab=1024, tied=1)
    P, C, B = 16, 16, 6
    lens = [40, 70, 23, 64, 90, 12, 55, 31, 77, 18, 44, 26, 61, 15]
    old = os.environ.get("OPPO_CHUNK_FLAGS")
    os.environ["OPPO_CHUNK_FLAGS"] = str(flags)
    try:
        eng = Engine(shape, dtype=abi.DTYPE_BF16, max_slots=16, max_prompt_len=P, max_response_len=96,
                     sample_seed=SAMPLE_SEED, carry=abi.CARRY_TOKEN, scorer_sms=scorer_sms)
    finally:
        if old is None:
            os.environ.pop("OPPO_CHUNK_FLAGS", None)
        else:
            os.environ["OPPO_CHUNK_FLAGS"] = old
    entries = list(S.seq_array(fresh_states(8, P, lens[:8])))
    eng.admit(entries)
    log, ro, nid = [], {}, 8
    for step in range(2):
        active = [e for e in entries if not e.scored]
        need = B - (len(entries) - len(active))
        outs, led = eng.run_step(active, C, abi.MODE_STREAMED, need)
        batch, entries, _ = S.select_finished(entries, outs, B)
        log.append(([o.as_tuple() for o in outs], led.score_us - led.decode_us))
        for b in batch:
            ro[b.id] = eng.read_rollout(b.id)
        eng.release([b.id for b in batch])
        fresh = list(S.seq_array(fresh_states(2, P, lens[nid:nid + 2], start_id=nid)))
        nid += 2
        eng.admit(fresh)
        entries = list(entries) + fresh
    eng.close()
    return log, ro


@pytest.mark.timeout(240, method="thread")
@pytest.mark.parametrize("scorer_sms", [0, 64])
def test_chunk_ready_flags_match_event_handoff(scorer_sms):
    """K13 on the device (north_star (2), engine.cpp:77-82): the actor stream
    publishes each wave's ready flag after the decode iteration that
    completes its chunks and the scorer stream's first kernel of the wave
    polls it -- every token, log-prob, value and reward is bit-identical to
    the per-wave event hand-off, with and without the SM partition (eager
    kernel loading, as conftest.py / bench.py set it)."""
    import os
    assert os.environ.get("CUDA_MODULE_LOADING") == "EAGER"
    la, ra = _run_flags(1, scorer_sms)
    lb, rb = _run_flags(0, scorer_sms)
    assert [x[0] for x in la] == [x[0] for x in lb]
    assert ra.keys() == rb.keys() and len(ra) >= 6
    for k in ra:
        for f in ("tokens", "old_lp", "ref_lp", "values"):
            assert np.array_equal(ra[k][f], rb[k][f]), (k, f)
        assert ra[k]["reward"] == rb[k]["reward"], k
    print("score tail after decode (us): flags", [x[1] for x in la], "events", [x[1] for x in lb])
