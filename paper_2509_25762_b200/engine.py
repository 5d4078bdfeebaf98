"""Python binding of the GPU step executor (liboppo.so engine entry points).

Mirrors the reference's executor interface: ``run_step`` (engine.hpp:91-93),
``select_finished``-compatible outcomes, ``ppo_update`` (fill_values +
toy_rlhf_step, ppo.cpp:274-317) and ``run_seed`` (driver.cpp:69-202).
"""
import ctypes as C

import numpy as np

from . import abi
from ._lib import check, lib
from .scheduler import seq_array

# Qwen2.5-family geometry; one vocabulary across all models.
VOCAB = 151936
SHAPES = {
    "tiny": dict(n_layers=2, d_model=128, n_heads=4, n_kv_heads=4, head_dim=32, d_ff=512,
                 vocab=512, tied=1),
    "0.5b": dict(n_layers=24, d_model=896, n_heads=14, n_kv_heads=2, head_dim=64, d_ff=4864,
                 vocab=VOCAB, tied=1),
    "1.5b": dict(n_layers=28, d_model=1536, n_heads=12, n_kv_heads=2, head_dim=128, d_ff=8960,
                 vocab=VOCAB, tied=1),
    "7b": dict(n_layers=28, d_model=3584, n_heads=28, n_kv_heads=4, head_dim=128, d_ff=18944,
               vocab=VOCAB, tied=0),
}
MODELS = ("actor", "reward", "critic", "ref")


def dims(shape):
    d = SHAPES[shape] if isinstance(shape, str) else shape
    return abi.ModelDims(**d)


def param_count(shape):
    d = SHAPES[shape] if isinstance(shape, str) else shape
    D, F, L = d["d_model"], d["d_ff"], d["n_layers"]
    qkv = (d["n_heads"] + 2 * d["n_kv_heads"]) * d["head_dim"]
    per = qkv * D + qkv + D * d["n_heads"] * d["head_dim"] + 3 * D * F + 2 * D
    emb = d["vocab"] * D * (1 if d["tied"] else 2)
    return L * per + emb + D


class Engine:
    def __init__(self, actor="tiny", reward=None, critic=None, ref=None, dtype=abi.DTYPE_BF16,
                 max_slots=16, max_prompt_len=8, max_response_len=64, page_size=64, kv_pages=0,
                 weight_seed=1, sample_seed=2, carry=abi.CARRY_CHUNK, train_heads=0, device=0,
                 nccl_comm=None, rank=0, world=1, use_graphs=1, scorer_sms=0, allreduce=None):
        cfg = abi.EngineCfg()
        cfg.actor = dims(actor)
        cfg.reward = dims(reward or actor)
        cfg.critic = dims(critic or reward or actor)
        cfg.ref = dims(ref or actor)
        cfg.dtype = dtype
        cfg.device = device
        cfg.weight_seed = weight_seed
        cfg.sample_seed = sample_seed
        cfg.max_slots = max_slots
        cfg.max_prompt_len = max_prompt_len
        cfg.max_response_len = max_response_len
        cfg.page_size = page_size
        cfg.kv_pages = kv_pages
        cfg.carry_granularity = carry
        cfg.rank, cfg.world = rank, world
        cfg.train_heads = train_heads
        cfg.use_graphs = use_graphs
        cfg.scorer_sms = scorer_sms
        cfg.nccl_comm = nccl_comm
        self._allreduce = None
        if allreduce is not None:  # host sum-allreduce (count, f64) over a device buffer
            def _cb(ctx, buf, count, dtype, stream):
                try:
                    allreduce(buf, count, bool(dtype), stream)
                    return 0
                except Exception:  # reported to the engine as a failed collective
                    return 1
            self._allreduce = ALLREDUCE_FN(_cb)
            cfg.allreduce = C.cast(self._allreduce, C.c_void_p)
        self.cfg = cfg
        self.h = C.c_void_p()
        check(lib().oppo_engine_create(C.byref(cfg), C.byref(self.h)))

    def close(self):
        if self.h:
            lib().oppo_engine_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        check(st, self.h)

    def admit(self, states, prompts=None):
        arr = seq_array(states)
        p = None
        if prompts is not None:
            flat = np.ascontiguousarray(np.concatenate([np.asarray(x) for x in prompts]),
                                        dtype=np.int32)
            p = flat.ctypes.data_as(C.POINTER(C.c_int32))
        self._check(lib().oppo_admit(self.h, arr, len(states), p))

    def run_step(self, active, chunk, mode, stop_after):
        arr = seq_array(active)
        out = (abi.SeqOutcome * max(1, len(active)))()
        led = abi.Ledger()
        self._check(lib().oppo_run_step(self.h, arr, len(active), chunk, mode, stop_after, out,
                                        C.byref(led)))
        return list(out[:len(active)]), led

    def ppo_update(self, ids, hp):
        arr = (C.c_int64 * max(1, len(ids)))(*ids)
        st = abi.PpoStats()
        self._check(lib().oppo_ppo_update(self.h, arr, len(ids), C.byref(hp), C.byref(st)))
        return st

    def save(self, path):
        """oppo_engine_save: slot table, KV pages, rollout buffers, trained heads."""
        L = lib()
        L.oppo_engine_save.argtypes = [C.c_void_p, C.c_char_p]
        self._check(L.oppo_engine_save(self.h, str(path).encode()))

    def load(self, path):
        """oppo_engine_load into this (fresh, same-configuration) engine."""
        L = lib()
        L.oppo_engine_load.argtypes = [C.c_void_p, C.c_char_p]
        self._check(L.oppo_engine_load(self.h, str(path).encode()))

    def release(self, ids):
        arr = (C.c_int64 * max(1, len(ids)))(*ids)
        self._check(lib().oppo_release(self.h, arr, len(ids)))

    def read_rollout(self, seq_id, cap=None):
        cap = cap or (self.cfg.max_response_len + 4)
        tok = (C.c_int32 * cap)()
        old = (C.c_float * cap)()
        ref = (C.c_float * cap)()
        val = (C.c_float * cap)()
        rew = C.c_float()
        n = C.c_int32()
        self._check(lib().oppo_read_rollout(self.h, seq_id, tok, old, ref, val, C.byref(rew), cap,
                                            C.byref(n)))
        L = n.value
        return dict(tokens=np.array(tok[1:L + 1]), old_lp=np.array(old[1:L + 1]),
                    ref_lp=np.array(ref[1:L + 1]), values=np.array(val[1:L + 1]),
                    reward=rew.value, length=L)

    def read_prompt(self, seq_id):
        cap = self.cfg.max_prompt_len
        out = (C.c_int32 * cap)()
        n = C.c_int32()
        L = lib()
        L.oppo_read_prompt.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int32), C.c_int32,
                                       C.POINTER(C.c_int32)]
        self._check(L.oppo_read_prompt(self.h, seq_id, out, cap, C.byref(n)))
        return list(out[:n.value])

    def get_tensor(self, model, name, layer=0):
        L = lib()
        L.oppo_get_tensor.argtypes = [C.c_void_p, C.c_int32, C.c_char_p, C.c_int32,
                                      C.POINTER(C.c_float), C.c_int64, C.POINTER(C.c_int64)]
        n = C.c_int64()
        self._check(L.oppo_get_tensor(self.h, model, name.encode(), layer, None, 0, C.byref(n)))
        if n.value == 0:
            return None
        buf = np.zeros(n.value, dtype=np.float32)
        self._check(L.oppo_get_tensor(self.h, model, name.encode(), layer,
                                      buf.ctypes.data_as(C.POINTER(C.c_float)), n.value,
                                      C.byref(n)))
        return buf

    def export_weights(self, model, masters=False):
        """fp32 copies of every tensor of one model (0 actor .. 3 ref), for the
        oracle; masters=True: the fp32 masters of the matrices the
        full-parameter update trains (where they exist)."""
        d = [self.cfg.actor, self.cfg.reward, self.cfg.critic, self.cfg.ref][model]
        mat = ("embed", "lm_head", "wqkv", "wo", "wgu", "wdown")
        nm = lambda k: k + ":master" if masters and k in mat else k
        w = {k: self.get_tensor(model, nm(k)) for k in ("embed", "lm_head", "final_norm", "head")}
        for k in ("ln1", "wqkv", "bqkv", "wo", "ln2", "wgu", "wdown"):
            w[k] = [self.get_tensor(model, nm(k), l) for l in range(d.n_layers)]
        dd = {f: getattr(d, f) for f, _ in abi.ModelDims._fields_}
        return dd, w

    def run_seed_ex(self, cfg, seed, prompt_fn=None, on_step=None):
        """oppo_run_seed_ex: the C++ step loop (driver.cpp:69-202) on this
        engine.  prompt_fn(id, prompt_len) -> tokens (host prompt source);
        on_step(record) -> truthy to stop.  Returns (records, selected ids per
        step, ledgers)."""
        def _pf(ctx, sid, plen, out):
            try:
                toks = prompt_fn(sid, plen)
                for i in range(plen):
                    out[i] = int(toks[i])
                return 0
            except Exception:
                return 1

        def _sf(ctx, rec):
            try:
                return 1 if on_step(rec.contents) else 0
            except Exception:
                return 1

        pf = abi.PROMPT_FN(_pf) if prompt_fn else None
        sf = abi.STEP_FN(_sf) if on_step else None
        leds = (abi.Ledger * cfg.steps)()
        hooks = abi.LoopHooks(C.cast(pf, C.c_void_p) if pf else None, None,
                              C.cast(sf, C.c_void_p) if sf else None, None, leds)
        recs = (abi.StepRecord * cfg.steps)()
        sel = (C.c_int64 * (cfg.steps * cfg.batch_size))()
        n = C.c_int32()
        self._check(lib().oppo_run_seed_ex(self.h, C.byref(cfg), seed, C.byref(hooks), recs, C.byref(n), sel))
        b = cfg.batch_size
        return (list(recs[:n.value]), [list(sel[i * b:(i + 1) * b]) for i in range(n.value)],
                list(leds[:n.value]))

    def run_seed(self, cfg, seed):
        recs = (abi.StepRecord * cfg.steps)()
        sel = (C.c_int64 * (cfg.steps * cfg.batch_size))()
        n = C.c_int32()
        self._check(lib().oppo_run_seed(self.h, C.byref(cfg), seed, recs, C.byref(n), sel))
        b = cfg.batch_size
        return list(recs[:n.value]), [list(sel[i * b:(i + 1) * b]) for i in range(n.value)]


NCCL_ID_BYTES = 128
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p)


def gloo_device_allreduce():
    """A host allreduce for oppo_engine_cfg.allreduce over the default
    torch.distributed (gloo) group: device -> host, all_reduce(SUM), host ->
    device (for CPU-transport tests of the data-parallel update)."""
    import torch
    import torch.distributed as dist
    cudart = C.CDLL("libcudart.so.12") if _have("libcudart.so.12") else C.CDLL("libcudart.so")
    cudart.cudaStreamSynchronize.argtypes = [C.c_void_p]
    cudart.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]

    def fn(buf, count, f64, stream):
        t = torch.empty(count, dtype=torch.float64 if f64 else torch.float32)
        nbytes = count * (8 if f64 else 4)
        assert cudart.cudaStreamSynchronize(stream) == 0
        assert cudart.cudaMemcpy(t.data_ptr(), buf, nbytes, 2) == 0  # device -> host
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        assert cudart.cudaMemcpy(buf, t.data_ptr(), nbytes, 1) == 0  # host -> device
        # a pageable host->device cudaMemcpy may return before its DMA lands, and
        # the engine's stream is non-blocking: wait for the copy explicitly
        assert cudart.cudaDeviceSynchronize() == 0
    return fn


def _have(name):
    try:
        C.CDLL(name)
        return True
    except OSError:
        return False


def nccl_comm_from_torch(rank, world, device):
    """One NCCL communicator for the engine (oppo_engine_cfg.nccl_comm): rank 0
    makes the id, torch.distributed (already initialised) broadcasts it."""
    import torch.distributed as dist
    buf = (C.c_uint8 * NCCL_ID_BYTES)()
    if rank == 0:
        check(lib().oppo_nccl_unique_id(buf))
    obj = [bytes(buf) if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    C.memmove(buf, obj[0], NCCL_ID_BYTES)
    comm = C.c_void_p()
    check(lib().oppo_nccl_comm_create(buf, world, rank, device, C.byref(comm)))
    return comm.value
