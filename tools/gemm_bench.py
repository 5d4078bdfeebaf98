import ctypes as C, sys
sys.path.insert(0, '.')
from paper_2509_25762_b200._lib import lib
L = lib()
shapes = [("lm_head decode M=282 LOGITS", 282, 151936, 896, 3, 3, 20),
          ("gate|up decode M=282 SWIGLU", 282, 9728, 896, 24, 2, 240),
          ("down decode M=282 ADDF32", 282, 896, 4864, 24, 1, 240),
          ("qkv decode M=256 STORE", 256, 1152, 896, 24, 0, 240),
          ("gate|up prefill M=8192 SWIGLU", 8192, 9728, 896, 4, 2, 20),
          ("gate|up decode M=64 SWIGLU", 64, 9728, 896, 24, 2, 240)]
for name, M, N, K, copies, epi, reps in shapes:
    us = C.c_float()
    st = L.oppo_k_gemm_bench(M, N, K, copies, reps, epi, C.byref(us))
    byts = N * K * 2 + M * K * 2
    fl = 2.0 * M * N * K
    if st != 0: print(name, "failed", L.oppo_last_error_global()); continue
    print(f"{name:32s} st={st} {us.value:9.2f} us  {byts/us.value/1e3:8.1f} GB/s  {fl/us.value/1e6:8.1f} TFLOP/s", flush=True)
