import sys, os, time
sys.path.insert(0, '.')
import numpy as np
from paper_2509_25762_b200 import abi, scheduler as S
from paper_2509_25762_b200.engine import Engine, SHAPES
layers = int(os.environ.get("LAYERS", "2")); B = int(os.environ.get("B", "16")); cap = int(os.environ.get("CAP", "128"))
steps = int(os.environ.get("STEPS", "3")); carry = int(os.environ.get("CARRY", "1")); MODE = int(os.environ.get("MODE", "0"))
shape = dict(SHAPES["0.5b"]); shape["n_layers"] = layers
P = 128; delta = max(1, B // 10); C = 64
eng = Engine(shape, shape, shape, shape, dtype=abi.DTYPE_BF16, max_slots=B + delta + 8, max_prompt_len=P, max_response_len=cap, train_heads=1, carry=carry)
lens = S.sample_lengths(abi.LengthDist(kind=1, mu_log=5.0, sigma_log=1.0, cap=cap), 7, 100000)
hp = abi.PpoHparams(gamma=1.0, lambda_=0.95, clip_epsilon=0.2, learning_rate=1e-3, value_learning_rate=1e-3, kl_coef=0.05, whiten=1)
entries, nid = [], 0
for step in range(steps):
    fresh = []
    while len(entries) + len(fresh) < B + delta:
        fresh.append(S.seq_array([dict(id=nid, prompt_len=P, target_len=lens[nid])])[0]); nid += 1
    eng.admit(fresh, prompts=[np.arange(P, dtype=np.int32) % 1000 + f.id for f in fresh])
    entries += fresh
    active = [e for e in entries if not e.scored]
    outs, led = eng.run_step(active, C, MODE, B - (len(entries) - len(active)))
    batch, entries, _ = S.select_finished(entries, outs, B)
    st = eng.ppo_update([b.id for b in batch], hp)
    eng.release([b.id for b in batch])
    print(f"step {step} wall {led.wall} step_ms {led.step_us/1e3:.1f} dec_ms {led.decode_us/1e3:.1f} sc_ms {led.score_us/1e3:.1f} pf_tok {led.prefill_tokens} upd_ms {st.update_us/1e3:.1f} obj {st.ppo_objective:.4f} R {st.mean_reward:.3f} kl {st.kl_mean:.4f} launches {led.kernel_launches}", flush=True)
