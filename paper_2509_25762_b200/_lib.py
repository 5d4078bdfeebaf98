"""Loads liboppo.so (built in-tree by ``make -C paper_2509_25762_b200/csrc``).

There is no fallback: if the shared library is missing the import fails loudly.
"""
import ctypes as C
import os

from . import abi

_HERE = os.path.dirname(os.path.abspath(__file__))
# OPPO_LIB: an alternative build of the same library (A/B perf comparisons)
LIB_PATH = os.environ.get("OPPO_LIB") or os.path.join(_HERE, "liboppo.so")

_lib = None


class OppoError(RuntimeError):
    """Raised for a non-zero oppo_status; ``code`` keeps the reference error class."""

    NAMES = {1: "ConfigError", 2: "InputError", 3: "InternalError", 4: "CudaError",
             5: "NcclError"}

    def __init__(self, code, msg):
        super().__init__(f"{self.NAMES.get(code, code)}: {msg}")
        self.code = code


class ConfigError(OppoError):
    pass


class InputError(OppoError):
    pass


class InternalError(OppoError):
    pass


def _raise(code, msg):
    cls = {1: ConfigError, 2: InputError, 3: InternalError}.get(code, OppoError)
    raise cls(code, msg)


def _preload_nccl():
    """liboppo.so links libnccl.so.2 by soname.  Load the NCCL that torch
    ships (pip nvidia-nccl, 2.28) first, so whichever of liboppo and torch is
    imported first, both bind to it: the system libnccl (2.27) lacks symbols
    libtorch_cuda needs (ncclDevCommCreate) and would break a later
    `import torch` if the loader picked it up for liboppo."""
    try:
        import nvidia.nccl as nn
    except ImportError:
        return
    for base in getattr(nn, "__path__", []):
        so = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(so):
            C.CDLL(so, mode=C.RTLD_GLOBAL)
            return


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run `make -C {_HERE}/csrc` "
                "(or __graft_entry__.build()). There is no CPU fallback.")
        _preload_nccl()
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
        _check_layout(_lib)
    return _lib


def check(status, engine=None):
    if status != 0:
        L = lib()
        if engine is not None:
            msg = L.oppo_last_error(engine).decode()
        else:
            msg = L.oppo_last_error_global().decode()
        _raise(status, msg)


def _declare(L):
    P = C.POINTER
    i32, i64, u64, dbl, vp = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_void_p
    sig = {
        "oppo_last_error_global": (C.c_char_p, []),
        "oppo_run_config_default": (None, [P(abi.RunConfig)]),
        "oppo_run_config_baseline": (None, [P(abi.RunConfig), P(abi.RunConfig)]),
        "oppo_run_config_validate": (i32, [P(abi.RunConfig)]),
        "oppo_rng_draws": (i32, [u64, C.c_char_p, i32, i64, vp]),
        "oppo_sample_lengths": (i32, [P(abi.LengthDist), u64, i64, P(i32)]),
        "oppo_build_schedule": (i32, [P(abi.SeqState), i32, i32, i32, P(abi.ChunkTask), i32,
                                      P(i32)]),
        "oppo_plan_step": (i32, [P(abi.SeqState), i32, i32, i32, i32, i32, P(abi.SeqOutcome),
                                 P(abi.Ledger)]),
        "oppo_select_finished": (i32, [P(abi.SeqState), i32, P(abi.SeqOutcome), i32, i32,
                                       P(abi.SeqState), P(i32), P(i32), P(i32)]),
        "oppo_delta_update": (i32, [i32, i32, i32, i32, i32, i32, P(dbl), P(i32), i32, P(i32),
                                    P(i32), P(dbl)]),
        "oppo_tuner_replay": (i32, [P(i32), i32, i32, P(i32), P(dbl), i32, P(i32)]),
        "oppo_abi_sizes": (i32, [P(i64), i32]),
        "oppo_run_seed_logical": (i32, [P(abi.RunConfig), u64, P(abi.StepRecord), P(i32),
                                        P(i64)]),
        "oppo_run_seed_logical_dp": (i32, [P(abi.RunConfig), u64, i32, i32, vp, vp, vp, vp,
                                           P(abi.StepRecord), P(i32), P(i64)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    # engine entry points (declared if present in the build)
    eng = {
        "oppo_engine_create": (i32, [P(abi.EngineCfg), P(vp)]),
        "oppo_engine_destroy": (None, [vp]),
        "oppo_last_error": (C.c_char_p, [vp]),
        "oppo_admit": (i32, [vp, P(abi.SeqState), i32, P(i32)]),
        "oppo_run_step": (i32, [vp, P(abi.SeqState), i32, i32, i32, i32, P(abi.SeqOutcome),
                                P(abi.Ledger)]),
        "oppo_ppo_update": (i32, [vp, P(i64), i32, P(abi.PpoHparams), P(abi.PpoStats)]),
        "oppo_release": (i32, [vp, P(i64), i32]),
        "oppo_read_rollout": (i32, [vp, i64, P(i32), P(C.c_float), P(C.c_float),
                                    P(C.c_float), P(C.c_float), i32, P(i32)]),
        "oppo_run_seed": (i32, [vp, P(abi.RunConfig), u64, P(abi.StepRecord), P(i32),
                                P(i64)]),
        "oppo_run_seed_ex": (i32, [vp, P(abi.RunConfig), u64, P(abi.LoopHooks), P(abi.StepRecord),
                                   P(i32), P(i64)]),
        "oppo_k_ppo_token": (i32, [i32, i32, vp, vp, vp, vp, vp, vp, dbl, dbl, dbl, i32, vp,
                                   vp, vp, vp, vp]),
        "oppo_k_gemm": (i32, [i32, i32, i32, i32, vp, vp, vp, vp, i32, vp]),
        "oppo_k_gemm_bench": (i32, [i32, i32, i32, i32, i32, i32, P(C.c_float)]),
        "oppo_k_gemm_t": (i32, [i32, i32, i32, i32, vp, i32, i32, vp, i32, i32, vp, i32, vp]),
        "oppo_k_gemm_dec": (i32, [i32, i32, i32, vp, vp, vp, vp, i32, vp, i64, P(i32), vp]),
        "oppo_nccl_unique_id": (i32, [vp]),
        "oppo_nccl_comm_create": (i32, [vp, i32, i32, i32, P(vp)]),
        "oppo_nccl_comm_destroy": (i32, [vp]),
    }
    for name, (res, args) in eng.items():
        f = getattr(L, name, None)
        if f is None:
            continue
        f.restype = res
        f.argtypes = args


def _check_layout(L):
    buf = (C.c_int64 * 32)()
    n = L.oppo_abi_sizes(buf, 32)
    want = list(abi.struct_sizes().values())
    got = list(buf[:n])
    if got != want:
        raise ImportError(f"liboppo.so ABI layout mismatch: C {got} vs ctypes {want}")
