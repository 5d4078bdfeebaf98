"""One full-parameter PPO update at the cfg2 shape (bench.py's engine), with
cudaProfilerStart/Stop around it so `ncu --profile-from-start off` captures
only the update.  Prints the update's device time."""
import ctypes as C
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import bench  # noqa: E402
from paper_2509_25762_b200 import abi  # noqa: E402
from paper_2509_25762_b200 import scheduler as S  # noqa: E402
from paper_2509_25762_b200.engine import Engine  # noqa: E402


def main():
    wl = bench.CFG2
    cfg = bench.make_cfg(wl)
    eng = Engine(wl["actor"], wl["scorer"], wl["scorer"], wl["scorer"], dtype=abi.DTYPE_BF16,
                 max_slots=wl["batch"] + wl["delta"] + 8, max_prompt_len=wl["prompt_len"],
                 max_response_len=wl["cap"], page_size=64, carry=cfg.carry_granularity,
                 train_heads=2, sample_seed=2, weight_seed=1, scorer_sms=56)
    V = eng.cfg.actor.vocab
    B, P = cfg.batch_size, cfg.prompt_len
    lengths = S.sample_lengths(cfg.lengths, 7, 4 * (B + cfg.delta_max))
    fresh = [S.seq_array([dict(id=i, prompt_len=P, target_len=lengths[i])])[0] for i in range(B + cfg.delta_init)]
    eng.admit(fresh, prompts=bench.host_prompts([f.id for f in fresh], P, V, 1234))
    outs, _ = eng.run_step(fresh, cfg.chunk_size, cfg.schedule_mode, B)
    batch, entries, _ = S.select_finished(fresh, outs, B)
    ids = [b.id for b in batch]
    hp = abi.PpoHparams(gamma=1.0, lambda_=0.95, clip_epsilon=0.2, learning_rate=1e-3,
                        value_learning_rate=1e-3, kl_coef=0.05, whiten=1)
    st = eng.ppo_update(ids, hp)  # warm (allocations, TMA maps)
    print("warm update_us", st.update_us, "tokens", st.n_tokens, flush=True)
    cudart = C.CDLL("libcudart.so.12")
    cudart.cudaProfilerStart()
    st = eng.ppo_update(ids, hp)
    cudart.cudaProfilerStop()
    print("update_us", st.update_us, "tokens", st.n_tokens, flush=True)
    eng.close()


if __name__ == "__main__":
    main()
