import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2509_25762_b200._lib import lib
L = lib()
def run(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    y = torch.full((M, N), float('nan'), device="cuda", dtype=torch.bfloat16)
    st = L.oppo_k_gemm(1, M, N, K, C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), None, C.c_void_p(y.data_ptr()), 0, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    ref = x.float() @ w.float().T
    d = (y.float() - ref).abs()
    bad = torch.isnan(y.float()) | (d > 0.05)
    rows = bad.any(1).nonzero().flatten().tolist()
    cols = bad.any(0).nonzero().flatten().tolist()
    print(M, N, K, "st", st, "bad rows", len(rows), rows[:5], rows[-5:] if rows else [], "bad cols", len(cols), cols[:4], cols[-4:] if cols else [], flush=True)
for M in [128, 144, 160, 240, 255, 257, 282, 300, 512, 700]:
    run(M, 256, 128)
