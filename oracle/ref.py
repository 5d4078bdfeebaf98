"""TEST INFRASTRUCTURE ONLY — ctypes binding of oracle/_ref/librlpipe_ref.so.

That library is the UNMODIFIED reference core (/root/reference/proj/core/src/*.cpp)
compiled by oracle/Makefile plus oracle/ref_shim.cpp.  Only tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference) may
import this module; the product package never does.
"""
import ctypes as C
import os

from paper_2509_25762_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "librlpipe_ref.so")
_ref = None


def available():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not available():
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C {HERE} ref`")
        L = C.CDLL(REF_SO)
        P = C.POINTER
        i32, i64, u64, dbl, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
        sigs = {
            "ref_last_error": (C.c_char_p, []),
            "ref_rng_draws": (i32, [u64, C.c_char_p, i32, i64, vp]),
            "ref_sample_lengths": (i32, [P(abi.LengthDist), u64, i64, P(i32)]),
            "ref_build_schedule": (i32, [P(abi.SeqState), i32, i32, i32, P(abi.ChunkTask), i32,
                                         P(i32)]),
            "ref_run_step": (i32, [P(abi.SeqState), i32, i32, i32, P(abi.Latency), i32,
                                   P(abi.SeqOutcome), P(abi.Ledger)]),
            "ref_select_finished": (i32, [P(abi.SeqState), i32, P(abi.SeqOutcome), i32, i32,
                                          P(abi.SeqState), P(i32), P(i32), P(i32)]),
            "ref_delta_update": (i32, [i32, i32, i32, i32, i32, i32, P(dbl), P(i32), i32,
                                       P(i32), P(i32), P(dbl)]),
            "ref_tuner_replay": (i32, [P(i32), i32, i32, P(i32), P(dbl), i32, P(i32)]),
            "ref_run_seed": (i32, [P(abi.RunConfig), u64, P(abi.StepRecord), P(i32), P(i32)]),
            "ref_run_seeds_parallel": (i32, [P(abi.RunConfig), P(u64), i32, P(i64)]),
            "ref_run_config_default": (i32, [P(abi.RunConfig)]),
            "ref_run_config_baseline": (i32, [P(abi.RunConfig), P(abi.RunConfig)]),
            "ref_write_outputs": (i32, [P(abi.RunConfig), P(u64), i32, C.c_char_p]),
            "ref_load_config": (i32, [C.c_char_p, C.c_char_p, C.c_char_p, i32, C.c_char_p, C.c_char_p,
                                      i32]),
            "ref_trace_seed": (i32, [P(abi.RunConfig), u64, P(abi.StepRecord), P(i32), P(i64),
                                     P(abi.SeqState), i32, P(i32)]),
            "ref_compute_gae": (i32, [P(dbl), P(dbl), i32, dbl, dbl, P(dbl)]),
            "ref_clipped_objective": (i32, [i32, P(dbl), i32, P(i32), P(i32), P(dbl), P(dbl),
                                            P(dbl), dbl, dbl, dbl, P(dbl), P(dbl)]),
            "ref_policy_logprobs": (i32, [i32, P(dbl), i32, P(dbl)]),
            "ref_rollouts": (i32, [i32, P(dbl), i32, dbl, dbl, u64, i32, P(i32), P(i32), P(dbl),
                                   P(dbl)]),
            "ref_toy_rlhf_step": (i32, [i32, i32, dbl, dbl, P(dbl), P(dbl), i32, P(i32), P(i32),
                                        P(dbl), P(dbl), dbl, dbl, dbl, dbl, dbl, P(dbl)]),
        }
        for name, (res, args) in sigs.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _ref = L
    return _ref


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


def rcheck(st):
    if st != 0:
        raise RefError(st, ref().ref_last_error().decode())


def rng_draws(seed, purpose, n, kind="u64"):
    ct = C.c_uint64 if kind == "u64" else C.c_double
    out = (ct * n)()
    rcheck(ref().ref_rng_draws(seed, purpose.encode(), {"u64": 0, "uniform01": 1,
                                                        "normal": 2}[kind], n, out))
    return list(out)


def sample_lengths(dist, seed, n):
    out = (C.c_int32 * n)()
    rcheck(ref().ref_sample_lengths(C.byref(dist), seed, n, out))
    return list(out)


def build_schedule(arr, n, chunk, mode=0):
    cap = 1 + sum(max(1, arr[i].target_len) for i in range(n)) + n
    tasks = (abi.ChunkTask * cap)()
    k = C.c_int32()
    rcheck(ref().ref_build_schedule(arr, n, chunk, mode, tasks, cap, C.byref(k)))
    return [(t.seq_id, t.first, t.last, t.index, bool(t.needs_decode)) for t in tasks[:k.value]]


def run_step(arr, n, chunk, mode, latency, stop_after):
    out = (abi.SeqOutcome * n)()
    led = abi.Ledger()
    rcheck(ref().ref_run_step(arr, n, chunk, mode, C.byref(latency), stop_after, out,
                              C.byref(led)))
    return list(out), led


def lockstep_latency():
    """The GPU executor's logical clock as a reference LatencyModel."""
    return abi.Latency(1, 0, 0, 0, 0, abi.PLACE_DISAGGREGATED, 1)


def run_seed(cfg, seed):
    recs = (abi.StepRecord * cfg.steps)()
    n, comp = C.c_int32(), C.c_int32()
    rcheck(ref().ref_run_seed(C.byref(cfg), seed, recs, C.byref(n), C.byref(comp)))
    return list(recs[:n.value]), bool(comp.value)


def write_outputs(cfg, seeds, out_dir):
    """rlpipe::run_experiment_in_memory + write_outputs into out_dir."""
    arr = (C.c_uint64 * len(seeds))(*seeds)
    rcheck(ref().ref_write_outputs(C.byref(cfg), arr, len(seeds), str(out_dir).encode()))


def trace_seed(cfg, seed, buf_cap=0):
    recs = (abi.StepRecord * cfg.steps)()
    sel = (C.c_int64 * (cfg.steps * cfg.batch_size))()
    n = C.c_int32()
    bufs = (abi.SeqState * max(1, cfg.steps * buf_cap))() if buf_cap else None
    counts = (C.c_int32 * cfg.steps)() if buf_cap else None
    rcheck(ref().ref_trace_seed(C.byref(cfg), seed, recs, C.byref(n), sel, bufs, buf_cap,
                                counts))
    b = cfg.batch_size
    out_bufs = None
    if buf_cap:
        out_bufs = [[bufs[i * buf_cap + j].as_tuple() for j in range(counts[i])]
                    for i in range(n.value)]
    return (list(recs[:n.value]), [list(sel[i * b:(i + 1) * b]) for i in range(n.value)],
            out_bufs)


def default_config(**overrides):
    """rlpipe::RunConfig{} (config.hpp:28-77) from the reference itself, with
    the same keyword overrides as scheduler.default_config; never touches
    liboppo.so (the reference arm of bench.py must not map the product)."""
    from paper_2509_25762_b200.scheduler import set_field  # pure ctypes field setter
    cfg = abi.RunConfig()
    rcheck(ref().ref_run_config_default(C.byref(cfg)))
    for k, v in overrides.items():
        set_field(cfg, k, v)
    return cfg


def baseline_config(cfg):
    """rlpipe::RunConfig::baseline (config.cpp:411-420) from the reference."""
    out = abi.RunConfig()
    rcheck(ref().ref_run_config_baseline(C.byref(cfg), C.byref(out)))
    return out


def run_seeds_parallel(cfg, seeds):
    arr = (C.c_uint64 * len(seeds))(*seeds)
    tot = C.c_int64()
    rcheck(ref().ref_run_seeds_parallel(C.byref(cfg), arr, len(seeds), C.byref(tot)))
    return tot.value


def ref_load_config(text):
    """rlpipe::load_config_text + config_echo + task_fingerprint + the echo of
    baseline(): dict(ok, echo, baseline_echo, fingerprint, error)."""
    cap = 1 << 16
    echo, base, fp, err = (C.create_string_buffer(cap), C.create_string_buffer(cap),
                           C.create_string_buffer(32), C.create_string_buffer(cap))
    st = ref().ref_load_config(text.encode("utf-8"), echo, base, cap, fp, err, cap)
    if st == 0:
        return dict(ok=True, echo=echo.value.decode(), baseline_echo=base.value.decode(),
                    fingerprint=fp.value.decode(), error="")
    return dict(ok=False, echo="", baseline_echo="", fingerprint="", error=err.value.decode(),
                config_error=st == 1)
