import sys, os, time
sys.path.insert(0, '.')
from paper_2509_25762_b200 import abi, scheduler as S
from paper_2509_25762_b200.engine import Engine, SHAPES
layers = int(os.environ.get("LAYERS", "2")); B = int(os.environ.get("B", "16")); cap = int(os.environ.get("CAP", "128"))
V = int(os.environ.get("V", "151936"))
shape = dict(SHAPES["0.5b"]); shape["n_layers"] = layers; shape["vocab"] = V
P = 128; delta = max(1, B // 10); C = 64
eng = Engine(shape, shape, shape, shape, dtype=abi.DTYPE_BF16, max_slots=B + delta + 8, max_prompt_len=P, max_response_len=cap, train_heads=1)
print("engine ok", flush=True)
lens = S.sample_lengths(abi.LengthDist(kind=1, mu_log=5.0, sigma_log=1.0, cap=cap), 7, 1000)
st = [dict(id=i, prompt_len=P, target_len=lens[i]) for i in range(B + delta)]
eng.admit(st); print("admit ok", flush=True)
t = time.time()
outs, led = eng.run_step(st, C, 0, B); print("step ok", led.wall, led.step_us, time.time() - t, flush=True)
batch, left, _ = S.select_finished(st, outs, B)
hp = abi.PpoHparams(gamma=1.0, lambda_=0.95, clip_epsilon=0.2, learning_rate=1e-3, value_learning_rate=1e-3, kl_coef=0.05, whiten=1)
import numpy as np
bad = {}
for b in st[:B]:
    try:
        ro = eng.read_rollout(b["id"])
    except Exception as ex:
        continue
    for k in ("old_lp", "ref_lp", "values"):
        if not np.all(np.isfinite(ro[k])):
            bad.setdefault(k, []).append((b["id"], int(np.sum(~np.isfinite(ro[k]))), ro["length"]))
    if not np.isfinite(ro["reward"]): bad.setdefault("reward", []).append(b["id"])
print("nonfinite:", {k: v[:5] for k, v in bad.items()}, flush=True)
ids_sel = [b.id for b in batch]
s2 = eng.ppo_update([b.id for b in batch], hp); print("update ok", s2.mean_reward, s2.ppo_objective, s2.update_us, flush=True)
for b in st[:4]:
    ro = eng.read_rollout(b["id"])
    idx = np.nonzero(~np.isfinite(ro["old_lp"]))[0]
    print(b["id"], "bad j:", (idx + 1).tolist(), "tokens:", ro["tokens"][idx].tolist(), "lp sample", ro["old_lp"][:6].tolist(), flush=True)
