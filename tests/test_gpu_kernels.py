"""Kernel-level GPU parity (run on a B200: pytest -m gpu).

GEMM: tcgen05/TMA bf16 path and SIMT fp32 path vs a torch fp32 reference.
PPO per-token kernels: fp64 vs the compiled reference's compute_gae /
clipped_objective (golden vectors), fp32 within stated tolerances.
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2509_25762_b200._lib import lib
    return lib()


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    torch.cuda.init()


EPI_STORE, EPI_ADD_F32, EPI_SWIGLU, EPI_STORE_F32 = 0, 1, 2, 5


@pytest.mark.parametrize("M,N,K", [(1, 128, 64), (7, 256, 128), (16, 896, 896), (33, 1152, 896),
                                   (100, 384, 4864), (256, 640, 256), (282, 1152, 896),
                                   (700, 512, 192), (2048, 896, 896)])
def test_gemm_bf16_tcgen05_vs_torch(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g)
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = _lib().oppo_k_gemm(1, M, N, K, _ptr(x), _ptr(w), _ptr(b), _ptr(y), EPI_STORE, _stream())
    assert st == 0, _lib().oppo_last_error_global()
    ref = x.float() @ w.float().T + b
    err = (y.float() - ref).abs().max().item()
    tol = 2e-2 * max(1.0, ref.abs().max().item())
    assert err <= tol, (err, tol)


@pytest.mark.parametrize("dtype", [1, 0])
@pytest.mark.parametrize("a_mn,b_mn", [(1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(896, 896, 1000), (1152, 4864, 640), (200, 136, 64), (4096, 896, 336)])
def test_gemm_mn_major_operands(dtype, a_mn, b_mn, M, N, K):
    """Operands read in place from their transposed storage (the update's
    wgrad dW = dY^T X with both MN-major over the token dimension, and dgrad
    dX = dY W with W MN-major): bit-identical to the K-major kernel on
    explicitly transposed copies (same tiles, same K order), and vs torch."""
    if dtype == 0 and M * N * K > 2e8:
        pytest.skip("SIMT path: small shapes only")
    tdt = torch.bfloat16 if dtype == 1 else torch.float32
    g = torch.Generator(device="cuda").manual_seed(M + 3 * N + 7 * K + a_mn + 2 * b_mn)
    a = torch.randn(M, K, device="cuda", generator=g).to(tdt)          # logical A [M][K]
    b = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(tdt)  # logical B [N][K]
    a_st = a.t().contiguous() if a_mn else a  # stored [K][M] when MN-major
    b_st = b.t().contiguous() if b_mn else b
    y = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    st = _lib().oppo_k_gemm_t(dtype, M, N, K, _ptr(a_st), a_mn, M if a_mn else K, _ptr(b_st), b_mn,
                              N if b_mn else K, _ptr(y), EPI_STORE_F32, _stream())
    assert st == 0, _lib().oppo_last_error_global()
    y_k = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    assert _lib().oppo_k_gemm_t(dtype, M, N, K, _ptr(a), 0, K, _ptr(b), 0, K, _ptr(y_k), EPI_STORE_F32,
                                _stream()) == 0
    assert torch.equal(y, y_k)
    ref = a.double() @ b.double().T
    rel = ((y.double() - ref).abs().max() / ref.abs().max()).item()
    assert rel < 2e-4, rel


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 1), (1, 0), (0, 1)])
def test_gemm_cta_pair_long_k(monkeypatch, a_mn, b_mn):
    """The long-K CTA-pair path (cta_group::2, 256x256 pair tiles, 6-stage
    ring; OPPO_TC2SM_LONGK=1) with K-major and MN-major operands: bit-identical
    across operand storage, within fp32-accumulation noise of float64, and
    equal to the single-CTA kernel up to accumulation order."""
    M, N, K = 2048, 8704, 4096
    g = torch.Generator(device="cuda").manual_seed(11 + a_mn + 2 * b_mn)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    a_st = a.t().contiguous() if a_mn else a
    b_st = b.t().contiguous() if b_mn else b

    def run(aa, am, bb, bm):
        y = torch.zeros(M, N, device="cuda", dtype=torch.float32)
        st = _lib().oppo_k_gemm_t(1, M, N, K, _ptr(aa), am, M if am else K, _ptr(bb), bm, N if bm else K,
                                  _ptr(y), EPI_STORE_F32, _stream())
        assert st == 0, _lib().oppo_last_error_global()
        return y

    monkeypatch.setenv("OPPO_TC2SM_LONGK", "1")
    y = run(a_st, a_mn, b_st, b_mn)
    y_k = run(a, 0, b, 0)
    assert torch.equal(y, y_k)
    ref = a.double() @ b.double().T
    rel = ((y.double() - ref).abs().max() / ref.abs().max()).item()
    assert rel < 2e-4, rel
    monkeypatch.setenv("OPPO_TC2SM_LONGK", "0")
    y1 = run(a, 0, b, 0)
    rel1 = ((y.double() - y1.double()).abs().max() / ref.abs().max()).item()
    assert rel1 < 2e-4, rel1


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1)])
def test_gemm_cta_pair_short_k(monkeypatch, a_mn, b_mn):
    """The short-K CTA-pair path (two pairs per SM pair, 3-stage ring;
    OPPO_TC2SM_SHORT=1) for the update's token-rich forward / dgrad GEMMs:
    within fp32-accumulation noise of float64 and of the single-CTA kernel."""
    M, N, K = 2048, 9728, 896
    g = torch.Generator(device="cuda").manual_seed(21 + b_mn)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    b_st = b.t().contiguous() if b_mn else b

    def run():
        y = torch.zeros(M, N, device="cuda", dtype=torch.float32)
        st = _lib().oppo_k_gemm_t(1, M, N, K, _ptr(a), a_mn, K, _ptr(b_st), b_mn, N if b_mn else K,
                                  _ptr(y), EPI_STORE_F32, _stream())
        assert st == 0, _lib().oppo_last_error_global()
        return y

    monkeypatch.setenv("OPPO_TC2SM_SHORT", "1")
    y = run()
    monkeypatch.setenv("OPPO_TC2SM_SHORT", "0")
    y1 = run()
    ref = a.double() @ b.double().T
    for out in (y, y1):
        rel = ((out.double() - ref).abs().max() / ref.abs().max()).item()
        assert rel < 2e-4, rel


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(2048, 896, 896), (1536, 4864, 896), (1104, 1152, 960)])
def test_gemm_persistent_update_path(monkeypatch, a_mn, b_mn, M, N, K):
    """The persistent double-buffered-TMEM GEMM as the PPO update uses it
    (OPPO_GEMM_PERSIST=2: 8 epilogue warps, K-major or MN-major operands,
    f32 store / f32 add epilogues): bit-identical to the 2-CTA/SM kernel
    (same tiles, same K order) and within fp32 noise of float64."""
    g = torch.Generator(device="cuda").manual_seed(M + N + a_mn + 2 * b_mn)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    a_st = a.t().contiguous() if a_mn else a
    b_st = b.t().contiguous() if b_mn else b
    y0 = torch.randn(M, N, device="cuda", generator=g)

    def run(epi):
        y = y0.clone()
        st = _lib().oppo_k_gemm_t(1, M, N, K, _ptr(a_st), a_mn, M if a_mn else K, _ptr(b_st), b_mn,
                                  N if b_mn else K, _ptr(y), epi, _stream())
        assert st == 0, _lib().oppo_last_error_global()
        return y

    for epi in (EPI_STORE_F32, EPI_ADD_F32):
        monkeypatch.setenv("OPPO_GEMM_PERSIST", "2")
        yp = run(epi)
        monkeypatch.setenv("OPPO_GEMM_PERSIST", "0")
        yt = run(epi)
        assert torch.equal(yp, yt), epi
        ref = a.double() @ b.double().T + (y0.double() if epi == EPI_ADD_F32 else 0)
        rel = ((yp.double() - ref).abs().max() / ref.abs().max()).item()
        assert rel < 2e-4, rel


def test_gemm_bf16_store_f32_long_k():
    # fp32 output isolates the tensor-core fp32 accumulation error over a long K
    M, N, K = 32, 256, 8192
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    y = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    st = _lib().oppo_k_gemm(1, M, N, K, _ptr(x), _ptr(w), None, _ptr(y), EPI_STORE_F32, _stream())
    assert st == 0
    ref = x.double() @ w.double().T
    rel = ((y.double() - ref).abs().max() / ref.abs().max()).item()
    assert rel < 2e-4, rel  # tensor-core fp32 accumulation (not IEEE-sequential)


def test_gemm_f32_simt_vs_torch():
    M, N, K = 37, 300, 96
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(M, K, device="cuda", generator=g)
    w = torch.randn(N, K, device="cuda", generator=g)
    y = torch.empty(M, N, device="cuda")
    assert _lib().oppo_k_gemm(0, M, N, K, _ptr(x), _ptr(w), None, _ptr(y), EPI_STORE, _stream()) == 0
    ref = x.double() @ w.double().T
    assert (y.double() - ref).abs().max().item() < 1e-4


def test_gemm_swiglu_epilogue():
    M, F, K = 50, 256, 128
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(2 * F, K, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    y = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    assert _lib().oppo_k_gemm(1, M, 2 * F, K, _ptr(x), _ptr(w), None, _ptr(y), EPI_SWIGLU, _stream()) == 0
    z = x.float() @ w.float().T
    gate, up = z[:, 0::2], z[:, 1::2]
    ref = torch.nn.functional.silu(gate) * up
    assert (y.float() - ref).abs().max().item() < 2e-2 * max(1, ref.abs().max().item())


@pytest.mark.parametrize("M,N,K,epi", [(4096, 9728, 896, EPI_SWIGLU), (8192, 4864, 896, EPI_STORE),
                                       (2304, 5120, 4864, EPI_STORE)])
def test_gemm_prefill_256x256_tile_vs_torch(M, N, K, epi, monkeypatch):
    """Token-rich GEMMs (prefill shapes) on the default 128x256-tile path."""
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.03).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g) if epi == EPI_STORE else None
    y = torch.empty(M, N // 2 if epi == EPI_SWIGLU else N, device="cuda", dtype=torch.bfloat16)
    st = _lib().oppo_k_gemm(1, M, N, K, _ptr(x), _ptr(w), _ptr(b) if b is not None else None, _ptr(y),
                            epi, _stream())
    assert st == 0, _lib().oppo_last_error_global()
    z = x.float() @ w.float().T
    ref = torch.nn.functional.silu(z[:, 0::2]) * z[:, 1::2] if epi == EPI_SWIGLU else z + b
    err = (y.float() - ref).abs().max().item()
    assert err <= 2e-2 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("persist", ["1", "0"])
@pytest.mark.parametrize("M,N,K,epi", [(1000, 896, 896, EPI_STORE), (8192, 9728, 896, EPI_SWIGLU),
                                       (3000, 1152, 896, EPI_STORE), (1025, 896, 4864, EPI_ADD_F32),
                                       (20000, 896, 896, EPI_STORE), (4100, 151936, 896, EPI_STORE)])
def test_gemm_prefill_persistent_vs_torch(M, N, K, epi, persist, monkeypatch):
    """Token-rich GEMMs on the persistent kernel (one CTA per SM, TMA ring,
    double-buffered TMEM accumulators; 128- or 256-wide tiles by N; ragged
    token counts, more tiles than SMs) and on the 2-CTA/SM tile kernel
    (OPPO_GEMM_PERSIST=0) against torch: SwiGLU / bias-store run on the
    persistent kernel, the residual add stays on the tile kernel."""
    monkeypatch.setenv("OPPO_GEMM_PERSIST", persist)
    g = torch.Generator(device="cuda").manual_seed(M + 3 * N + K)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.03).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g) if epi == EPI_STORE else None
    if epi == EPI_ADD_F32:
        y0 = torch.randn(M, N, device="cuda", generator=g)
        y = y0.clone()
    else:
        y = torch.empty(M, N // 2 if epi == EPI_SWIGLU else N, device="cuda", dtype=torch.bfloat16)
    st = _lib().oppo_k_gemm(1, M, N, K, _ptr(x), _ptr(w), _ptr(b) if b is not None else None, _ptr(y),
                            epi, _stream())
    assert st == 0, _lib().oppo_last_error_global()
    torch.cuda.synchronize()
    z = x.float() @ w.float().T
    if epi == EPI_SWIGLU:
        ref = torch.nn.functional.silu(z[:, 0::2]) * z[:, 1::2]
    elif epi == EPI_ADD_F32:
        ref = y0 + z
    else:
        ref = z + b
    err = (y.float() - ref).abs().max().item()
    assert err <= 2e-2 * max(1.0, ref.abs().max().item()), err


# decode GEMM (swap-AB tcgen05, gemm_dec.cuh): partial sums over splits, SwiGLU, store+bias
@pytest.mark.parametrize("M,N,K", [(1, 128, 64), (16, 1152, 896), (40, 896, 896), (64, 896, 4864),
                                   (129, 384, 256), (256, 896, 4864), (282, 1152, 896),
                                   (298, 896, 4864), (512, 256, 128)])
def test_gemm_dec_partials_vs_torch(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 11 + N)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    ws_floats = 16 << 20
    ws = torch.full((ws_floats,), float("nan"), device="cuda")
    sp = C.c_int32(0)
    st = _lib().oppo_k_gemm_dec(M, N, K, _ptr(x), _ptr(w), None, None, 0, _ptr(ws), ws_floats,
                                C.byref(sp), _stream())
    assert st == 0, _lib().oppo_last_error_global()
    assert 1 <= sp.value <= K // 64
    y = ws[: sp.value * M * N].view(sp.value, M, N).sum(0)  # every partial written (no NaN left)
    ref = x.double() @ w.double().T
    rel = ((y.double() - ref).abs().max() / ref.abs().max()).item()
    assert rel < 1e-4, rel


@pytest.mark.parametrize("M", [3, 64, 200, 282])
def test_gemm_dec_swiglu_and_store(M):
    F, K = 384, 896
    g = torch.Generator(device="cuda").manual_seed(M)
    x = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(2 * F, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    b = torch.randn(2 * F, device="cuda", generator=g)
    y = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    assert _lib().oppo_k_gemm_dec(M, 2 * F, K, _ptr(x), _ptr(w), None, _ptr(y), 1, None, 0, None,
                                  _stream()) == 0
    z = x.float() @ w.float().T
    ref = torch.nn.functional.silu(z[:, 0::2]) * z[:, 1::2]
    assert (y.float() - ref).abs().max().item() < 2e-2 * max(1, ref.abs().max().item())
    y2 = torch.empty(M, 2 * F, device="cuda", dtype=torch.bfloat16)
    assert _lib().oppo_k_gemm_dec(M, 2 * F, K, _ptr(x), _ptr(w), _ptr(b), _ptr(y2), 2, None, 0, None,
                                  _stream()) == 0
    ref2 = z + b
    assert (y2.float() - ref2).abs().max().item() < 2e-2 * max(1, ref2.abs().max().item())


# ------------------------------------------------------------------ PPO
def _ragged(case_list, key):
    return np.concatenate([np.asarray(c[key], dtype=np.float64) for c in case_list])


def test_gae_fp64_bit_exact_vs_reference(golden):
    cases = golden["gae"]
    L = _lib()
    for c in cases:
        T = len(c["rewards"])
        off = torch.tensor([0, T], dtype=torch.int32, device="cuda")
        rew = torch.tensor(c["rewards"], dtype=torch.float64, device="cuda")
        val = torch.tensor(c["values"], dtype=torch.float64, device="cuda")
        adv = torch.empty(T, dtype=torch.float64, device="cuda")
        ret = torch.empty(T, dtype=torch.float64, device="cuda")
        st = L.oppo_k_ppo_token(1, 1, _ptr(off), None, _ptr(rew), _ptr(val), None, None, c["gamma"],
                                c["lambda"], 0.2, 0, _ptr(adv), _ptr(ret), None, None, _stream())
        assert st == 0
        got = adv.cpu().numpy()
        assert np.array_equal(got, np.asarray(c["adv"])), (got, c["adv"])


def test_gae_fp32_scan_within_tolerance(golden):
    L = _lib()
    cases = golden["gae"]
    offs = [0]
    for c in cases:
        offs.append(offs[-1] + len(c["rewards"]))
    # one batched launch, one warp per sequence; gamma/lambda per batch -> use the first case's
    g0, l0 = cases[0]["gamma"], cases[0]["lambda"]
    rew = np.concatenate([c["rewards"] for c in cases])
    vals = np.concatenate([c["values"] for c in cases])
    off = torch.tensor(offs, dtype=torch.int32, device="cuda")
    r = torch.tensor(rew, dtype=torch.float32, device="cuda")
    v = torch.tensor(vals, dtype=torch.float32, device="cuda")
    adv = torch.empty(len(rew), dtype=torch.float32, device="cuda")
    ret = torch.empty(len(rew), dtype=torch.float32, device="cuda")
    assert L.oppo_k_ppo_token(0, len(cases), _ptr(off), None, _ptr(r), _ptr(v), None, None, g0, l0,
                              0.2, 0, _ptr(adv), _ptr(ret), None, None, _stream()) == 0
    got = adv.cpu().numpy()
    # fp64 oracle of the same recursion (compute_gae, ppo.cpp:71-85)
    want = []
    for i, c in enumerate(cases):
        run = 0.0
        out = []
        T = len(c["rewards"])
        for t in range(T - 1, -1, -1):
            d = c["rewards"][t] + g0 * c["values"][t + 1] - c["values"][t]
            run = d + g0 * l0 * run
            out.append(run)
        want.extend(out[::-1])
    want = np.asarray(want)
    assert np.max(np.abs(got - want) / np.maximum(1, np.abs(want))) < 1e-5


def test_clipped_objective_fp64_vs_reference(golden):
    L = _lib()
    for c in golden["clipped"]:
        offs = c["offsets"]
        n = len(offs) - 1
        N = offs[-1]
        off = torch.tensor(offs, dtype=torch.int32, device="cuda")
        score = torch.tensor(c["rewards"], dtype=torch.float64, device="cuda")
        vals = torch.tensor(c["values"], dtype=torch.float64, device="cuda")
        new = torch.tensor(c["new_lp"], dtype=torch.float64, device="cuda")
        old = torch.tensor(c["old_lp"], dtype=torch.float64, device="cuda")
        adv = torch.empty(N, dtype=torch.float64, device="cuda")
        ret = torch.empty(N, dtype=torch.float64, device="cuda")
        dobj = torch.empty(N, dtype=torch.float64, device="cuda")
        osum = torch.zeros(1, dtype=torch.float64, device="cuda")
        st = L.oppo_k_ppo_token(1, n, _ptr(off), _ptr(score), None, _ptr(vals), _ptr(new), _ptr(old),
                                c["gamma"], c["lambda"], c["eps"], 0, _ptr(adv), _ptr(ret),
                                _ptr(dobj), _ptr(osum), _stream())
        assert st == 0
        obj = osum.item() / N
        assert abs(obj - c["objective"]) <= 1e-12 * max(1, abs(c["objective"]))
        # table gradient from the per-token dObj/dlogp (clipped_objective_grad, ppo.cpp:138-177)
        V = c["vocab"]
        theta = np.asarray(c["theta"]).reshape(V + 1, V)
        grad = np.zeros_like(theta)
        d = dobj.cpu().numpy()
        for i in range(n):
            prev = 0
            for t in range(offs[i], offs[i + 1]):
                row = theta[prev]
                p = np.exp(row - row.max())
                p /= p.sum()
                e = np.zeros(V)
                e[c["tokens"][t]] = 1
                grad[prev] += d[t] * (e - p)
                prev = c["tokens"][t] + 1
        ref = np.asarray(c["grad"]).reshape(V + 1, V)
        assert np.max(np.abs(grad - ref)) < 1e-12
