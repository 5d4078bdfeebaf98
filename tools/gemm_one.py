"""One GEMM shape through oppo_k_gemm_bench, for ncu captures.
env: M N K EPI (0 store, 1 add f32, 2 swiglu, 3 logits) REPS"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25762_b200._lib import lib  # noqa: E402

e = {k: int(os.environ.get(k, d)) for k, d in dict(M=8192, N=9728, K=896, EPI=2, REPS=3, COPIES=2).items()}
us = C.c_float()
st = lib().oppo_k_gemm_bench(e["M"], e["N"], e["K"], e["COPIES"], e["REPS"], e["EPI"], C.byref(us))
print(e, "status", st, f"{us.value:.2f} us", f"{2.0 * e['M'] * e['N'] * e['K'] / us.value / 1e6:.1f} TFLOP/s")
