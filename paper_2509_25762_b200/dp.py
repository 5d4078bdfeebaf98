"""Data-parallel OPPO step loop, one process per GPU.

Each rank runs the reference's step loop (driver.cpp:103-195) on its own
prompt shard: its own overcommit buffer of B/N + delta/N entries, its own
length stream ``Rng::derive(seed ^ rank, "lengths")``, its own generation,
scoring, selection and KV carry — no collective on the data path.  The only
exchange is the per-step statistics allreduce: {sum reward, n samples} (plus
the whitening moments and the head gradients, which the GPU engine reduces
inside ``oppo_ppo_update`` over NCCL).  Every rank feeds the GLOBAL mean
reward to an identical DeltaController (overcommit.hpp:81), so all ranks take
the same delta decisions.

The executor is pluggable: ``GpuExecutor`` (the B200 engine) or
``LogicalExecutor`` (the same decisions on the CPU, used by the gloo tests).
"""
import ctypes as C
import time

import numpy as np

from . import abi
from . import scheduler as S


class LogicalExecutor:
    """run_step on the lockstep logical clock (no GPU); reward = reward_fn(id)."""

    def __init__(self, carry=abi.CARRY_CHUNK, reward_fn=None):
        self.carry = carry
        self.reward_fn = reward_fn or (lambda i: float(i % 7) / 7.0)

    def admit(self, fresh, prompts=None):
        return 0

    def run_step(self, active, chunk, mode, stop_after):
        return S.plan_step(active, chunk, mode, stop_after, self.carry)

    def update(self, ids, hp):
        r = [self.reward_fn(i) for i in ids]
        return {"sum_reward": float(sum(r)), "n": len(ids), "global": False}

    def release(self, ids):
        pass


class GpuExecutor:
    """The B200 engine (engine.Engine); with an NCCL communicator its
    ppo_update already returns the global mean reward."""

    def __init__(self, engine, prompt_fn=None):
        self.eng = engine
        self.prompt_fn = prompt_fn

    def admit(self, fresh, prompts=None):
        if prompts is None and self.prompt_fn is not None:
            prompts = self.prompt_fn([f.id for f in fresh])
        self.eng.admit(fresh, prompts=prompts)
        return sum(np.asarray(p).nbytes for p in prompts) if prompts is not None else 0

    def run_step(self, active, chunk, mode, stop_after):
        return self.eng.run_step(active, chunk, mode, stop_after)

    def update(self, ids, hp):
        st = self.eng.ppo_update(ids, hp) if ids else abi.PpoStats()
        glob = self.eng.cfg.world > 1 and bool(self.eng.cfg.nccl_comm)
        return {"sum_reward": st.mean_reward * (1 if glob else len(ids)), "n": 1 if glob else len(ids),
                "global": glob, "stats": st}

    def release(self, ids):
        self.eng.release(ids)


def run_rank(cfg, seed, rank, world, executor, allreduce_sum=None, steps=None, on_step=None):
    """Runs `steps` OPPO steps of one rank.  allreduce_sum(list[float]) ->
    list[float] sums across ranks (None: single rank).  Returns per-step dicts
    with the selected ids, delta, global mean reward and the executor's
    ledger."""
    B = cfg.batch_size
    steps = cfg.steps if steps is None else steps
    lengths = S.sample_lengths(cfg.lengths, seed ^ rank, max(1024, (B + cfg.delta_max + 1) * (steps + 2)))
    ctl = S.DeltaController(cfg.controller, cfg.window, cfg.delta_min, cfg.delta_max, cfg.delta_inc,
                            cfg.delta_dec)
    entries, next_id, delta = [], 0, cfg.delta_init
    out = []
    for step in range(steps):
        t0 = time.perf_counter()
        fresh = []
        while len(entries) + len(fresh) < B + delta:  # refill (overcommit.cpp:11-28)
            gid = next_id * world + rank  # rank r serves prompt ids = r (mod N)
            fresh.append(S.seq_array([dict(id=gid, prompt_len=cfg.prompt_len,
                                           target_len=lengths[next_id], admitted_at=step,
                                           arrival_step=step)])[0])
            next_id += 1
        h2d = executor.admit(fresh) if fresh else 0
        h2d += len(fresh) * C.sizeof(abi.SeqState)
        entries = entries + fresh
        active = [e for e in entries if not e.scored]
        need = B - (len(entries) - len(active))  # pre-scored entries count first (driver.cpp:129-145)
        outs, led = [], abi.Ledger()
        if active and need > 0:
            outs, led = executor.run_step(active, cfg.chunk_size, cfg.schedule_mode, need)
            h2d += len(active) * C.sizeof(abi.SeqState)
        batch, entries, _ = S.select_finished(entries, outs, B)
        ids = [b.id for b in batch]
        upd = executor.update(ids, cfg.ppo)
        executor.release(ids)
        if upd["global"] or allreduce_sum is None or world == 1:
            mean = upd["sum_reward"] / max(1, upd["n"])
        else:
            s, n = allreduce_sum([upd["sum_reward"], float(upd["n"])])
            mean = s / max(1.0, n)
        ctl.observe(mean)
        delta, _ = ctl.update(delta)
        rec = dict(step=step, ids=ids, delta=delta, mean_reward=mean, ledger=led, outs=outs,
                   stats=upd.get("stats"), h2d=h2d, wall_s=time.perf_counter() - t0,
                   d2h=len(outs) * C.sizeof(abi.SeqOutcome) + C.sizeof(abi.PpoStats) + len(ids) * 8)
        out.append(rec)
        if on_step:
            on_step(rec)
    return out


def run_lockstep_oracle(cfg, seed, world, reward_fn=None, steps=None):
    """N rank buffers stepped in lockstep in ONE process with one shared
    controller fed the global mean (SURVEY 8e's oracle at N ranks)."""
    steps = cfg.steps if steps is None else steps
    B = cfg.batch_size
    ex = LogicalExecutor(cfg.carry_granularity, reward_fn)
    lengths = [S.sample_lengths(cfg.lengths, seed ^ r, max(1024, (B + cfg.delta_max + 1) * (steps + 2)))
               for r in range(world)]
    ctl = S.DeltaController(cfg.controller, cfg.window, cfg.delta_min, cfg.delta_max, cfg.delta_inc,
                            cfg.delta_dec)
    entries = [[] for _ in range(world)]
    nxt = [0] * world
    delta = cfg.delta_init
    hist = [[] for _ in range(world)]
    for step in range(steps):
        tot, cnt = 0.0, 0
        for r in range(world):
            while len(entries[r]) < B + delta:
                gid = nxt[r] * world + r
                entries[r].append(S.seq_array([dict(id=gid, prompt_len=cfg.prompt_len,
                                                    target_len=lengths[r][nxt[r]], admitted_at=step,
                                                    arrival_step=step)])[0])
                nxt[r] += 1
            active = [e for e in entries[r] if not e.scored]
            need = B - (len(entries[r]) - len(active))
            outs = []
            if active and need > 0:
                outs, _ = ex.run_step(active, cfg.chunk_size, cfg.schedule_mode, need)
            batch, entries[r], _ = S.select_finished(entries[r], outs, B)
            ids = [b.id for b in batch]
            u = ex.update(ids, cfg.ppo)
            tot += u["sum_reward"]
            cnt += u["n"]
            hist[r].append(ids)
        ctl.observe(tot / max(1, cnt))
        delta, _ = ctl.update(delta)
        for r in range(world):
            hist[r][-1] = (hist[r][-1], delta)
    return hist
