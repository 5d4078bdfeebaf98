"""Decode/prefill GEMM sweep through oppo_k_gemm_bench (CUDA events, distinct
weight copies so weights stream from HBM).  Prints us, weight GB/s, TFLOP/s."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25762_b200._lib import lib  # noqa: E402

L = lib()
# name, N, K, copies, epilogue (0 store, 1 add f32, 2 swiglu, 3 logits)
SHAPES = [("qkv", 1152, 896, 24, 0), ("o", 896, 896, 24, 1), ("gate|up", 9728, 896, 24, 2),
          ("down", 896, 4864, 24, 1), ("lm_head", 151936, 896, 3, 3)]
if os.environ.get("SHAPE") == "7b":  # 7B actor (cfg4 / cfg5) decode projections
    SHAPES = [("qkv", 4608, 3584, 3, 0), ("o", 3584, 3584, 3, 1), ("gate|up", 37888, 3584, 3, 2),
              ("down", 3584, 18944, 3, 1)]
if os.environ.get("DEC", "1") == "1":  # decode GEMM (gemm_dec): 16 partials, 17 SwiGLU
    SHAPES = [(n, N, K, c, {0: 16, 1: 16, 2: 17}.get(e, e)) for n, N, K, c, e in SHAPES]
if os.environ.get("PREFILL") == "1":  # scorer prefill pass shapes (token-tiled kernels)
    SHAPES = [("qkv", 1152, 896, 4, 0), ("o", 896, 896, 4, 1), ("gate|up", 9728, 896, 4, 2),
              ("down", 896, 4864, 4, 1)]
Ms = [int(x) for x in os.environ.get("MS", "16,64,128,282").split(",")]
tot = {}
for M in Ms:
    for name, N, K, copies, epi in SHAPES:
        us = C.c_float()
        reps = 30 if epi == 3 else 240
        st = L.oppo_k_gemm_bench(M, N, K, copies, reps, epi, C.byref(us))
        if st != 0:
            print(name, M, "failed", L.oppo_last_error_global())
            continue
        byts = N * K * 2 + M * K * 2
        fl = 2.0 * M * N * K
        mult = 1 if name == "lm_head" else (28 if os.environ.get("SHAPE") == "7b" else 24)
        tot[M] = tot.get(M, 0.0) + mult * us.value
        print(f"M={M:4d} {name:8s} {us.value:9.2f} us {byts/us.value/1e3:8.1f} GB/s "
              f"{fl/us.value/1e6:8.1f} TFLOP/s", flush=True)
for M, t in tot.items():
    print(f"M={M}: GEMM time per decode iteration (24 layers + lm_head) {t/1e3:.3f} ms; "
          f"HBM floor {0.988e9/6.55e12*1e3:.3f} ms")
