"""Python mirror of the reference's scheduler interface, backed by liboppo.so.

Names and argument meanings follow rlpipe (``/root/reference/proj/core``):
``build_schedule`` (chunking.cpp:20-48), ``run_step`` on the GPU's logical
clock (engine.cpp:24-223 under the lockstep latency model), ``select_finished``
(overcommit.cpp:30-95), ``DeltaController.update`` (overcommit.cpp:134-155),
``retune`` (chunking.cpp:73-100) and ``run_seed`` (driver.cpp:69-202).
Errors raise ConfigError / InputError / InternalError like the reference.
"""
import ctypes as C

from . import abi
from ._lib import check, lib

_DRAW_KIND = {"u64": 0, "uniform01": 1, "normal": 2}


def default_config(**overrides):
    """RunConfig{} defaults (config.hpp:28-77) with keyword overrides.

    Nested fields use ``latency_*``, ``lengths_*`` and ``ppo_*`` prefixes, e.g.
    ``lengths_kind=abi.LEN_LOGNORMAL, lengths_mu_log=5.0``; ``chunk_candidates``
    takes a list.
    """
    cfg = abi.RunConfig()
    lib().oppo_run_config_default(C.byref(cfg))
    for k, v in overrides.items():
        set_field(cfg, k, v)
    return cfg


def set_field(cfg, key, value):
    if key == "chunk_candidates":
        cfg.n_candidates = len(value)
        for i, x in enumerate(value):
            cfg.chunk_candidates[i] = x
        return
    if key == "lengths_table":
        cfg.lengths.table_n = len(value)
        for i, (ln, w) in enumerate(value):
            cfg.lengths.table_len[i] = ln
            cfg.lengths.table_w[i] = w
        return
    for prefix, sub in (("latency_", "latency"), ("lengths_", "lengths"), ("ppo_", "ppo")):
        if key.startswith(prefix):
            name = key[len(prefix):]
            if sub == "ppo" and name == "lambda":
                name = "lambda_"
            setattr(getattr(cfg, sub), name, value)
            return
    setattr(cfg, key, value)


def baseline(cfg):
    """RunConfig::baseline (config.cpp:411-420)."""
    out = abi.RunConfig()
    lib().oppo_run_config_baseline(C.byref(cfg), C.byref(out))
    return out


def validate(cfg):
    check(lib().oppo_run_config_validate(C.byref(cfg)))


def rng_draws(seed, purpose, n, kind="u64"):
    ct = C.c_uint64 if kind == "u64" else C.c_double
    out = (ct * n)()
    check(lib().oppo_rng_draws(seed, purpose.encode(), _DRAW_KIND[kind], n, out))
    return list(out)


def sample_lengths(dist, seed, n):
    out = (C.c_int32 * n)()
    check(lib().oppo_sample_lengths(C.byref(dist), seed, n, out))
    return list(out)


def seq_array(states):
    arr = (abi.SeqState * max(1, len(states)))()
    for i, s in enumerate(states):
        if isinstance(s, abi.SeqState):
            arr[i] = s
        else:
            for k, v in s.items():
                setattr(arr[i], k, v)
    return arr


def build_schedule(states, chunk_size, mode=abi.MODE_STREAMED):
    arr = seq_array(states)
    cap = sum(max(1, s.target_len) for s in arr[:len(states)]) + len(states) + 1
    tasks = (abi.ChunkTask * cap)()
    n = C.c_int32()
    check(lib().oppo_build_schedule(arr, len(states), chunk_size, mode, tasks, cap, C.byref(n)))
    return [(t.seq_id, t.first, t.last, t.index, bool(t.needs_decode)) for t in tasks[:n.value]]


def plan_step(states, chunk_size, mode, stop_after, carry=abi.CARRY_CHUNK):
    arr = seq_array(states)
    out = (abi.SeqOutcome * len(states))()
    led = abi.Ledger()
    check(lib().oppo_plan_step(arr, len(states), chunk_size, mode, stop_after, carry, out,
                               C.byref(led)))
    return list(out), led


def select_finished(entries, outcomes, batch_size):
    arr = seq_array(entries)
    outs = (abi.SeqOutcome * max(1, len(outcomes)))(*outcomes)
    sel = (abi.SeqState * max(1, len(entries)))()
    nb, nr, sb = C.c_int32(), C.c_int32(), C.c_int32()
    check(lib().oppo_select_finished(arr, len(entries), outs, len(outcomes), batch_size, sel,
                                     C.byref(nb), C.byref(nr), C.byref(sb)))
    return list(sel[:nb.value]), list(arr[:nr.value]), bool(sb.value)


class DeltaController:
    """DeltaController (overcommit.hpp:71-90)."""

    def __init__(self, mode=abi.DELTA_ALG1, window=8, delta_min=0, delta_max=8, inc=1, dec=1):
        self.mode, self.window = mode, window
        self.delta_min, self.delta_max, self.inc, self.dec = delta_min, delta_max, inc, dec
        self.reward_history = []

    def observe(self, r):
        self.reward_history.append(r)

    def update(self, delta):
        n = len(self.reward_history)
        hist = (C.c_double * max(1, n))(*self.reward_history)
        nh, nd, hs, st = C.c_int32(n), C.c_int32(), C.c_int32(), C.c_double()
        check(lib().oppo_delta_update(self.mode, self.window, self.delta_min, self.delta_max,
                                      self.inc, self.dec, hist, C.byref(nh), delta, C.byref(nd),
                                      C.byref(hs), C.byref(st)))
        self.reward_history = list(hist[:nh.value])
        return nd.value, (st.value if hs.value else None)


def tuner_replay(candidates, window, measurements):
    n = len(measurements)
    cand = (C.c_int32 * len(candidates))(*candidates)
    mc = (C.c_int32 * max(1, n))(*[m[0] for m in measurements])
    mv = (C.c_double * max(1, n))(*[m[1] for m in measurements])
    chosen = (C.c_int32 * max(1, n))()
    check(lib().oppo_tuner_replay(cand, len(candidates), window, mc, mv, n, chosen))
    return list(chosen[:n])


def run_seed_logical(cfg, seed):
    """run_seed (driver.cpp:69-202) with the GPU's logical executor, no GPU work.

    Returns (records, selected ids per step)."""
    recs = (abi.StepRecord * cfg.steps)()
    sel = (C.c_int64 * (cfg.steps * cfg.batch_size))()
    n = C.c_int32()
    check(lib().oppo_run_seed_logical(C.byref(cfg), seed, recs, C.byref(n), sel))
    b = cfg.batch_size
    return list(recs[:n.value]), [list(sel[i * b:(i + 1) * b]) for i in range(n.value)]


def run_seed_logical_dp(cfg, seed, rank, world, allreduce_sum=None, batch_reward=None):
    """The C++ step loop (driver.hpp) as rank `rank` of `world` on the logical
    executor: allreduce_sum(list[float]) -> list[float] sums over the ranks;
    batch_reward(ids) -> the selected batch's mean reward (simulate mode).
    Returns (records, selected ids per step)."""
    def _ar(ctx, v, n):
        try:
            out = allreduce_sum([v[i] for i in range(n)])
            for i in range(n):
                v[i] = out[i]
            return 0
        except Exception:
            return 1

    def _rw(ctx, ids, n):
        return float(batch_reward([ids[i] for i in range(n)]))

    ar = abi.HOST_ALLREDUCE_FN(_ar) if allreduce_sum else None
    rw = abi.BATCH_REWARD_FN(_rw) if batch_reward else None
    recs = (abi.StepRecord * cfg.steps)()
    sel = (C.c_int64 * (cfg.steps * cfg.batch_size))()
    n = C.c_int32()
    check(lib().oppo_run_seed_logical_dp(C.byref(cfg), seed, rank, world,
                                         C.cast(ar, C.c_void_p) if ar else None, None,
                                         C.cast(rw, C.c_void_p) if rw else None, None,
                                         recs, C.byref(n), sel))
    b = cfg.batch_size
    return list(recs[:n.value]), [list(sel[i * b:(i + 1) * b]) for i in range(n.value)]
