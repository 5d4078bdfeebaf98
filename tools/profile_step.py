"""One cfg2-shaped OPPO step for ncu launch lists (not a bench: numbers taken
under a profiler are never reported as bench values).

  MODE=1 (sequential) puts the actor decode iterations first, then one scorer
  wave, so per-kernel shares of a decode iteration read cleanly.
  env: B (256), CAP (1024), STEPS (1), MODE (1), LAYERS (24)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2509_25762_b200 import abi, scheduler as S
from paper_2509_25762_b200.engine import Engine, SHAPES

B = int(os.environ.get("B", "256"))
CAP = int(os.environ.get("CAP", "1024"))
STEPS = int(os.environ.get("STEPS", "1"))
MODE = int(os.environ.get("MODE", "1"))
shape = dict(SHAPES["0.5b"])
shape["n_layers"] = int(os.environ.get("LAYERS", "24"))
P, C, delta = 128, 64, B // 10
eng = Engine(shape, shape, shape, shape, dtype=abi.DTYPE_BF16, max_slots=B + delta + 8,
             max_prompt_len=P, max_response_len=CAP, train_heads=1, carry=abi.CARRY_TOKEN)
lens = S.sample_lengths(abi.LengthDist(kind=1, mu_log=5.0, sigma_log=1.0, cap=CAP), 7, 100000)
hp = abi.PpoHparams(gamma=1.0, lambda_=0.95, clip_epsilon=0.2, learning_rate=1e-3,
                    value_learning_rate=1e-3, kl_coef=0.05, whiten=1)
entries, nid = [], 0
for step in range(STEPS):
    fresh = []
    while len(entries) + len(fresh) < B + delta:
        fresh.append(S.seq_array([dict(id=nid, prompt_len=P, target_len=lens[nid])])[0])
        nid += 1
    eng.admit(fresh, prompts=[np.arange(P, dtype=np.int32) % 1000 + f.id for f in fresh])
    entries += fresh
    active = [e for e in entries if not e.scored]
    outs, led = eng.run_step(active, C, MODE, B - (len(entries) - len(active)))
    batch, entries, _ = S.select_finished(entries, outs, B)
    st = eng.ppo_update([b.id for b in batch], hp)
    eng.release([b.id for b in batch])
    print(f"step {step} iters {led.decode_iters} dec_ms {led.decode_us/1e3:.1f} "
          f"sc_ms {led.score_us/1e3:.1f} upd_ms {st.update_us/1e3:.1f}", flush=True)
eng.close()
