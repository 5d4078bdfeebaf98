"""Data-parallel host logic on CPU (gloo, world_size 2).

Two processes each run one rank of the OPPO step loop (paper_2509_25762_b200.dp)
on the logical executor: own prompt shard (ids = r mod N), own length stream
Rng::derive(seed ^ r, "lengths"), statistics allreduced over gloo, one Delta
controller per rank fed the global mean.  Checked against the in-process
lockstep oracle (N buffers, one shared controller): identical selections and
identical delta trajectories on every rank.
"""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _cfg():
    from paper_2509_25762_b200 import abi
    from paper_2509_25762_b200 import scheduler as S
    return S.default_config(
        mode=abi.RUN_SIMULATE, steps=12, batch_size=6, prompt_len=4, delta_init=3, delta_min=0,
        delta_max=6, controller=abi.DELTA_ALG1, window=2, chunk_size=8,
        schedule_mode=abi.MODE_STREAMED, carry_granularity=abi.CARRY_CHUNK,
        lengths_kind=abi.LEN_LOGNORMAL, lengths_mu_log=3.0, lengths_sigma_log=0.8, lengths_cap=64,
        latency_decode_per_token=1, latency_prefill_per_token=0, latency_reward_residual=0,
        latency_placement=abi.PLACE_DISAGGREGATED)


def _reward(i):
    return float((i * 2654435761) % 97) / 97.0


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_25762_b200 import dp

    def allreduce_sum(vals):
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.tolist()

    cfg = _cfg()
    recs = dp.run_rank(cfg, 11, rank, world, dp.LogicalExecutor(cfg.carry_granularity, _reward),
                       allreduce_sum)
    q.put((rank, [(r["ids"], r["delta"], r["mean_reward"]) for r in recs]))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_gloo_matches_lockstep_oracle():
    from paper_2509_25762_b200 import dp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = _cfg()
    oracle = dp.run_lockstep_oracle(cfg, 11, world, _reward)
    deltas = {tuple(d for _, d, _ in got[r]) for r in range(world)}
    assert len(deltas) == 1, "ranks took different delta decisions"
    assert len(set(next(iter(deltas)))) > 1, "controller never moved: test is vacuous"
    for r in range(world):
        assert [ids for ids, _, _ in got[r]] == [ids for ids, _ in oracle[r]]
        assert [d for _, d, _ in got[r]] == [d for _, d in oracle[r]]
        assert all(i % world == r for ids, _, _ in got[r] for i in ids)  # prompt shard
    # the two ranks see different length streams (seed ^ rank), so different work
    assert got[0][0][0] != [i - 1 for i in got[1][0][0]]


def test_single_rank_matches_oracle_world1():
    from paper_2509_25762_b200 import dp
    cfg = _cfg()
    recs = dp.run_rank(cfg, 5, 0, 1, dp.LogicalExecutor(cfg.carry_granularity, _reward))
    oracle = dp.run_lockstep_oracle(cfg, 5, 1, _reward)
    assert [r["ids"] for r in recs] == [ids for ids, _ in oracle[0]]


def _worker_cpp(rank, world, port, q):
    """The same rank through the C++ step loop (driver.hpp, oppo_run_seed_logical_dp)."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_25762_b200 import scheduler as S

    def allreduce_sum(vals):
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.tolist()

    def batch_reward(ids):
        return sum(_reward(i) for i in ids) / len(ids) if ids else 0.0

    cfg = _cfg()
    recs, sel = S.run_seed_logical_dp(cfg, 11, rank, world, allreduce_sum, batch_reward)
    q.put((rank, [(ids, r.delta, r.mean_reward) for ids, r in zip(sel, recs)]))
    dist.destroy_process_group()


def test_two_rank_cpp_loop_matches_lockstep_oracle():
    """The production loop in C++ (rank/world, seed ^ rank lengths, prompt ids
    = r mod N, global mean reward into every rank's controller): identical
    selections and Delta trajectories to the in-process lockstep oracle."""
    from paper_2509_25762_b200 import dp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_cpp, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = _cfg()
    oracle = dp.run_lockstep_oracle(cfg, 11, world, _reward)
    assert len({tuple(d for _, d, _ in got[r]) for r in range(world)}) == 1
    for r in range(world):
        assert [[i for i in ids if i >= 0] for ids, _, _ in got[r]] == [ids for ids, _ in oracle[r]]
        # StepRecord.delta is the step's capacity; the oracle logs the updated one
        assert [d for _, d, _ in got[r]][1:] == [d for _, d in oracle[r]][:-1]
        assert all(i % world == r for ids, _, _ in got[r] for i in ids if i >= 0)
    # global mean reward: both ranks record the same value each step
    assert [m for _, _, m in got[0]] == [m for _, _, m in got[1]]
