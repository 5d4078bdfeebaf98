"""A small streamed OPPO step for compute-sanitizer (memcheck / racecheck /
synccheck): 0.5B width, 2 layers, bf16, overcommitted streamed step with the
scorer partition and three scorer streams, then the full-parameter update.
  compute-sanitizer --tool racecheck python tools/sanitize_step.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25762_b200 import abi, scheduler as S  # noqa: E402
from paper_2509_25762_b200.engine import Engine  # noqa: E402

shape = dict(n_layers=2, d_model=896, n_heads=14, n_kv_heads=2, head_dim=64, d_ff=4864, vocab=1024, tied=1)
P, C, B = 16, 16, 4
lens = [40, 21, 33, 12, 28, 19]
eng = Engine(shape, dtype=abi.DTYPE_BF16, max_slots=8, max_prompt_len=P, max_response_len=48,
             sample_seed=3, carry=abi.CARRY_TOKEN, train_heads=2,
             scorer_sms=int(os.environ.get("SCORER_SMS", "64")))
st = list(S.seq_array([dict(id=i, prompt_len=P, target_len=L) for i, L in enumerate(lens)]))
eng.admit(st)
outs, led = eng.run_step(st, C, abi.MODE_STREAMED, B)
batch, left, _ = S.select_finished(st, outs, B)
hp = abi.PpoHparams(gamma=1.0, lambda_=0.95, clip_epsilon=0.2, learning_rate=1e-3, value_learning_rate=1e-3,
                    kl_coef=0.05, whiten=1)
stats = eng.ppo_update([b.id for b in batch], hp)
eng.release([b.id for b in batch])
eng.close()
print("sanitize step ok", led.wall, stats.n_tokens, flush=True)
