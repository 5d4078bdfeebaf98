"""Data-parallel PPO update across two ranks, on one GPU.

Two processes (gloo process group) each own a shard of the prompts and an
engine on cuda:0; their oppo_ppo_update reduces {whitening moments, token
count, reward sum} and the lm_head / value-head gradients through the
engine's allreduce hook (here a gloo host allreduce; NCCL in production, same
call sites).  After one step both ranks must hold the same heads, equal (fp32
tolerance) to ONE engine updating on the union batch, and report the global
mean reward.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


@pytest.fixture(autouse=True)
def _one_attention_split(monkeypatch):
    """One attention split for every batch size: identical per-row decode
    arithmetic on the 4-row shards and the 8-row union (row-independent fp32
    path).  Set per test (spawned ranks inherit it), not at import, so the
    other modules of the session keep the default split rule."""
    monkeypatch.setenv("OPPO_ATTN_MAX_SPLIT", "1")
LENS = [9, 14, 5, 20, 11, 7, 16, 12]
P, CHUNK = 8, 8


def _hp():
    from paper_2509_25762_b200 import abi
    return abi.PpoHparams(gamma=1.0, lambda_=0.95, clip_epsilon=0.2, learning_rate=0.5,
                          value_learning_rate=0.3, kl_coef=0.05, whiten=1)


def _run(ids, rank, world, allreduce, train=1, nccl=None):
    from paper_2509_25762_b200 import abi
    from paper_2509_25762_b200.engine import Engine
    eng = Engine("tiny", dtype=abi.DTYPE_F32, max_slots=8, max_prompt_len=P, max_response_len=32,
                 sample_seed=2, train_heads=train, rank=rank, world=world, allreduce=allreduce,
                 nccl_comm=nccl)
    states = [dict(id=i, prompt_len=P, target_len=LENS[i]) for i in ids]
    eng.admit(states)
    eng.run_step(states, CHUNK, abi.MODE_STREAMED, len(states))
    toks = {i: eng.read_rollout(i)["tokens"].tolist() for i in ids}
    st = eng.ppo_update(ids, _hp())
    out = dict(lm=eng.get_tensor(0, "lm_head").copy(), vh=eng.get_tensor(2, "head").copy(),
               reward=st.mean_reward, tokens=st.n_tokens, obj=st.ppo_objective, toks=toks)
    if train == 2:  # trunk tensors of the full-parameter update
        for m in (0, 2):
            for k in ("wqkv", "wgu", "wdown", "ln1"):
                out[f"{m}.{k}"] = eng.get_tensor(m, k, 1).copy()
    eng.close()
    return out


def _worker(rank, world, port, q, train=1):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2509_25762_b200.engine import gloo_device_allreduce
    ids = [i for i in range(len(LENS)) if i % world == rank]
    q.put((rank, _run(ids, rank, world, gloo_device_allreduce(), train)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("train", [1, 2], ids=["heads", "full"])
def test_two_rank_update_equals_union_batch_update(train):
    """train=2: the full-parameter update's per-tensor gradient allreduce."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, train)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    single = _run(list(range(len(LENS))), 0, 1, None, train)
    for r in range(2):  # same rollouts on the shards as in the union batch
        for i, t in got[r]["toks"].items():
            assert t == single["toks"][i], (r, i)
    for r in range(2):
        for k in [k for k in single if k in ("lm", "vh") or "." in k]:
            a, b = got[r][k], single[k]
            assert np.max(np.abs(a - b)) <= 1e-5 * max(1.0, np.abs(b).max()), (r, k)
        assert abs(got[r]["reward"] - single["reward"]) < 1e-9
    # the update moved the weights (the comparison is not vacuous)
    from paper_2509_25762_b200 import abi
    from paper_2509_25762_b200.engine import Engine
    e0 = Engine("tiny", dtype=abi.DTYPE_F32, max_slots=8, max_prompt_len=P, max_response_len=32,
                sample_seed=2, train_heads=1)
    w0 = e0.get_tensor(0, "lm_head").copy()
    e0.close()
    assert np.max(np.abs(single["lm"] - w0)) > 1e-6


def _nccl_world1(q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    os.environ["MASTER_PORT"] = str(s.getsockname()[1])
    s.close()
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_2509_25762_b200._lib import lib
    from paper_2509_25762_b200.engine import nccl_comm_from_torch
    comm = nccl_comm_from_torch(0, 1, 0)
    ids = list(range(len(LENS)))
    with_nccl = _run(ids, 0, 1, None, 2, comm)
    plain = _run(ids, 0, 1, None, 2, None)
    lib().oppo_nccl_comm_destroy(comm)
    dist.destroy_process_group()
    q.put({k: bool(np.array_equal(with_nccl[k], plain[k])) for k in with_nccl if k != "toks"})


def test_nccl_call_sites_on_hardware_world1():
    """The engine's NCCL call sites (whitening / reward statistics, and the
    full-parameter update's per-layer gradient buckets: grouped allreduce +
    SGD on a comm stream overlapped with the rest of the backward) executed
    on the GPU with a world-1 communicator: the update is bit-identical to
    the engine without one, whose SGD runs after the backward on the compute
    stream (the sum over one rank is the identity)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_world1, args=(q,))
    p.start()
    same = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert all(same.values()), same
