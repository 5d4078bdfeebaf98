"""TMA streaming probe: aggregate GB/s of pure TMA box loads (no compute) vs
CTAs, pipeline depth and box size, from a 128 MB matrix (> L2)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_25762_b200._lib import lib  # noqa: E402

L = lib()
f = L.oppo_k_tma_probe
f.restype = C.c_int32
f.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_float), C.POINTER(C.c_float)]
for ctas in (76, 148, 296):
    for stages in (4, 8, 12):
        for box_rows in (128, 256):
            if stages * box_rows * 128 > 200 * 1024:
                continue
            per = max(stages * 4, (128 << 20) // (box_rows * 128) // ctas)
            us, gbs = C.c_float(), C.c_float()
            st = f(ctas, stages, box_rows, per, C.byref(us), C.byref(gbs))
            print(f"ctas={ctas:4d} stages={stages:3d} box={box_rows * 128 // 1024:3d} KB: "
                  f"{gbs.value:8.1f} GB/s ({us.value:.1f} us)" if st == 0 else f"fail {st}", flush=True)
