"""TEST INFRASTRUCTURE ONLY — ctypes binding of oracle/liboppo_oracle.so, the
plain-C restatement of the reference's hot path (see oppo_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it.
"""
import ctypes as C
import os

import numpy as np

from paper_2509_25762_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboppo_oracle.so")
_L = None


def lib():
    global _L
    if _L is None:
        if not os.path.exists(SO):
            raise FileNotFoundError(f"{SO} missing: run `make -C {HERE} oracle`")
        L = C.CDLL(SO)
        P = C.POINTER
        i32, i64, u64, dbl, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
        L.oracle_rng_draws.argtypes = [u64, C.c_char_p, C.c_int, i64, vp]
        L.oracle_sample_lengths.argtypes = [P(abi.LengthDist), u64, i64, P(i32)]
        L.oracle_run_step.argtypes = [P(abi.SeqState), C.c_int, C.c_int, C.c_int, P(abi.Latency),
                                      C.c_int, C.c_int, P(abi.SeqOutcome), P(abi.Ledger)]
        L.oracle_run_seed.argtypes = [P(abi.RunConfig), u64, P(i64), P(i64), P(C.c_int)]
        L.oracle_gae.argtypes = [P(dbl), P(dbl), C.c_int, dbl, dbl, P(dbl)]
        L.oracle_ppo_clip.argtypes = [C.c_int, P(dbl), P(dbl), P(dbl), dbl, P(dbl)]
        L.oracle_ppo_clip.restype = dbl
        L.oracle_gpt_forward.argtypes = [vp, P(i32), C.c_int, P(dbl), P(dbl)]
        L.oracle_token_key.argtypes = [u64, i64, i32]
        L.oracle_token_key.restype = u64
        L.oracle_gumbel.argtypes = [u64, C.c_uint32]
        L.oracle_gumbel.restype = C.c_float
        L.oracle_sample_token.argtypes = [P(dbl), C.c_int, u64, P(dbl), P(dbl), P(dbl)]
        L.oracle_sample_token.restype = C.c_int
        L.oracle_prompt_token.argtypes = [u64, i64, i32, i32]
        L.oracle_prompt_token.restype = i32
        _L = L
    return _L


def rng_draws(seed, purpose, n, kind="u64"):
    ct = C.c_uint64 if kind == "u64" else C.c_double
    out = (ct * n)()
    lib().oracle_rng_draws(seed, purpose.encode(), {"u64": 0, "uniform01": 1, "normal": 2}[kind],
                           n, out)
    return list(out)


def sample_lengths(dist, seed, n):
    out = (C.c_int32 * n)()
    lib().oracle_sample_lengths(C.byref(dist), seed, n, out)
    return list(out)


def run_step(arr, n, chunk, mode, latency, stop_after, credit_partial=False):
    out = (abi.SeqOutcome * n)()
    led = abi.Ledger()
    lib().oracle_run_step(arr, n, chunk, mode, C.byref(latency), stop_after, int(credit_partial),
                          out, C.byref(led))
    return list(out), led


def run_seed(cfg, seed):
    rec = (C.c_int64 * (4 * cfg.steps))()
    sel = (C.c_int64 * (cfg.steps * cfg.batch_size))()
    n = C.c_int()
    lib().oracle_run_seed(C.byref(cfg), seed, rec, sel, C.byref(n))
    b = cfg.batch_size
    return ([tuple(rec[4 * i:4 * i + 4]) for i in range(n.value)],
            [list(sel[i * b:(i + 1) * b]) for i in range(n.value)])


def gae(rewards, values, gamma, lam):
    T = len(rewards)
    out = (C.c_double * T)()
    lib().oracle_gae((C.c_double * T)(*rewards), (C.c_double * (T + 1))(*values), T, gamma, lam,
                     out)
    return list(out)


def ppo_clip(new_lp, old_lp, adv, eps):
    n = len(new_lp)
    D = C.c_double * n
    d = D()
    obj = lib().oracle_ppo_clip(n, D(*new_lp), D(*old_lp), D(*adv), eps, d)
    return obj, list(d)


class _Gpt(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("d", C.c_int), ("H", C.c_int), ("KV", C.c_int),
                ("hd", C.c_int), ("dff", C.c_int), ("V", C.c_int),
                ("embed", C.c_void_p), ("lm_head", C.c_void_p), ("final_norm", C.c_void_p),
                ("ln1", C.c_void_p), ("wqkv", C.c_void_p), ("bqkv", C.c_void_p),
                ("wo", C.c_void_p), ("ln2", C.c_void_p), ("wgu", C.c_void_p),
                ("wdown", C.c_void_p)]


class GptOracle:
    """fp64 forward of one model on float32 weight arrays (dict from the engine export)."""

    def __init__(self, dims, w):
        self.dims, self.w = dims, w
        L = dims["n_layers"]
        self._keep = []

        def arr(x):
            a = np.ascontiguousarray(x, dtype=np.float32)
            self._keep.append(a)
            return a.ctypes.data

        def ptrs(name):
            p = (C.c_void_p * L)(*[arr(w[name][l]) for l in range(L)])
            self._keep.append(p)
            return C.cast(p, C.c_void_p)

        self.s = _Gpt(L, dims["d_model"], dims["n_heads"], dims["n_kv_heads"], dims["head_dim"],
                      dims["d_ff"], dims["vocab"], arr(w["embed"]), arr(w["lm_head"]),
                      arr(w["final_norm"]), ptrs("ln1"), ptrs("wqkv"), ptrs("bqkv"), ptrs("wo"),
                      ptrs("ln2"), ptrs("wgu"), ptrs("wdown"))

    def forward(self, tokens, logits=True):
        T = len(tokens)
        d, V = self.dims["d_model"], self.dims["vocab"]
        hid = np.zeros((T, d), dtype=np.float64)
        lg = np.zeros((T, V), dtype=np.float64) if logits else None
        tok = np.ascontiguousarray(tokens, dtype=np.int32)
        lib().oracle_gpt_forward(C.byref(self.s), tok.ctypes.data_as(C.POINTER(C.c_int32)), T,
                                 hid.ctypes.data_as(C.POINTER(C.c_double)),
                                 lg.ctypes.data_as(C.POINTER(C.c_double)) if logits else None)
        return hid, lg


def token_key(seed, seq, pos):
    return lib().oracle_token_key(seed, seq, pos)


def gumbel_row(key, V):
    g = lib().oracle_gumbel
    return np.array([g(key, v) for v in range(V)], dtype=np.float32)


def sample_token(logits, key):
    """(token, log-prob, block margin, in-block margin) of the engine's two-level draw."""
    x = np.ascontiguousarray(logits, dtype=np.float64)
    lp, mb, mi = C.c_double(), C.c_double(), C.c_double()
    tok = lib().oracle_sample_token(x.ctypes.data_as(C.POINTER(C.c_double)), len(x), key,
                                    C.byref(lp), C.byref(mb), C.byref(mi))
    return tok, lp.value, mb.value, mi.value


def prompt_tokens(seed, seq_id, P, V):
    f = lib().oracle_prompt_token
    return [f(seed, seq_id, q, V) for q in range(P)]
