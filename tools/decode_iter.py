"""Actor decode-iteration time at a constant batch M (0.5B actor, bf16):
admit M sequences of equal length L, run one sequential-mode step (every
iteration decodes all M rows), report decode_loop_us / L and the decode
loop's algorithmic HBM bytes rate.  Second run of each M (graph captured)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2509_25762_b200 import abi, scheduler as S
from paper_2509_25762_b200.engine import Engine, SHAPES

Ms = [int(x) for x in os.environ.get("MS", "16,64,128,256").split(",")]
L, P = int(os.environ.get("L", "48")), int(os.environ.get("P", "128"))  # P: context before the first decode
SHAPE = os.environ.get("SHAPE", "0.5b")
shape = dict(SHAPES[SHAPE])
eng = Engine(shape, shape, shape, shape, dtype=abi.DTYPE_BF16, max_slots=max(Ms) + 8, max_prompt_len=P,
             max_response_len=L, train_heads=0, carry=abi.CARRY_TOKEN,
             use_graphs=int(os.environ.get("GRAPHS", "1")))
PROFILE = os.environ.get("PROFILE") == "1"  # cudaProfilerStart/Stop around the graph-captured run
if PROFILE:
    import ctypes
    cudart = ctypes.CDLL("libcudart.so.12")
nid = 0
for M in Ms:
    for rep in range(2):
        seqs = S.seq_array([dict(id=nid + i, prompt_len=P, target_len=L) for i in range(M)])
        nid += M
        eng.admit(seqs, prompts=[(np.arange(P, dtype=np.int32) * 7 + s.id) % 1000 for s in seqs])
        if PROFILE and rep == 1:
            cudart.cudaProfilerStart()
        outs, led = eng.run_step(list(seqs), 64, abi.MODE_SEQUENTIAL, M)
        if PROFILE and rep == 1:
            cudart.cudaProfilerStop()
        eng.release([s.id for s in seqs])
    per = led.decode_loop_us / L
    gbs = (led.decode_weight_bytes + led.decode_kv_bytes) / (led.decode_loop_us * 1e-6) / 1e9
    print(f"M={M:4d} decode iteration {per:8.1f} us  alg {gbs:7.1f} GB/s  "
          f"alg_bytes_per_iteration {(led.decode_weight_bytes + led.decode_kv_bytes) / L:.0f}  "
          f"(weights {led.decode_weight_bytes / L / 1e6:.0f} MB + KV {led.decode_kv_bytes / L / 1e6:.1f} MB "
          f"per iteration)", flush=True)
eng.close()
