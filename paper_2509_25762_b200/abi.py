"""ctypes mirror of include/oppo/oppo.h (the C ABI of liboppo.so).

Field order and types follow the header exactly; tests check sizeof parity
through ``oppo_abi_sizes`` exported by the library.
"""
import ctypes as C

OPPO_OK, OPPO_ERR_CONFIG, OPPO_ERR_INPUT, OPPO_ERR_INTERNAL, OPPO_ERR_CUDA, OPPO_ERR_NCCL = range(6)
MODE_STREAMED, MODE_SEQUENTIAL = 0, 1
PLACE_COLOCATED, PLACE_DISAGGREGATED = 0, 1
LEN_TWO_POINT, LEN_LOGNORMAL, LEN_EMPIRICAL = 0, 1, 2
DELTA_FIXED, DELTA_ALG1, DELTA_EQ4 = 0, 1, 2
RUN_SIMULATE, RUN_TRAIN, RUN_TUNE = 0, 1, 2
CARRY_CHUNK, CARRY_TOKEN = 0, 1
DTYPE_F32, DTYPE_BF16 = 0, 1
MAX_TABLE = 64
MAX_CANDIDATES = 16


class SeqState(C.Structure):
    _fields_ = [("id", C.c_int64), ("prompt_len", C.c_int32), ("arrival_step", C.c_int32),
                ("target_len", C.c_int32), ("generated", C.c_int32),
                ("prefilled_tokens", C.c_int32), ("chunks_emitted", C.c_int32),
                ("chunks_prefilled", C.c_int32), ("finished", C.c_int32), ("scored", C.c_int32),
                ("admitted_at", C.c_int32), ("deferrals", C.c_int32), ("_pad", C.c_int32)]

    def as_tuple(self):
        return tuple(getattr(self, f) for f, _ in self._fields_ if f != "_pad")


class ChunkTask(C.Structure):
    _fields_ = [("seq_id", C.c_int64), ("first", C.c_int32), ("last", C.c_int32),
                ("index", C.c_int32), ("needs_decode", C.c_int32)]


class SeqOutcome(C.Structure):
    _fields_ = [("seq_id", C.c_int64), ("score_ready", C.c_int64),
                ("tokens_decoded", C.c_int32), ("tokens_prefilled", C.c_int32),
                ("decode_chunks_completed", C.c_int32), ("prefill_tasks_completed", C.c_int32),
                ("carry_prefill_completed", C.c_int32), ("_pad", C.c_int32)]

    def as_tuple(self):
        return tuple(getattr(self, f) for f, _ in self._fields_ if f != "_pad")


class Ledger(C.Structure):
    _fields_ = [("wall", C.c_int64), ("busy_generation", C.c_int64), ("busy_scoring", C.c_int64),
                ("work_generation", C.c_int64), ("work_scoring", C.c_int64),
                ("step_us", C.c_double), ("decode_us", C.c_double), ("score_us", C.c_double),
                ("decode_iters", C.c_int64), ("decode_tokens", C.c_int64),
                ("prefill_tokens", C.c_int64), ("kernel_launches", C.c_int64),
                ("decode_loop_us", C.c_double), ("decode_weight_bytes", C.c_double),
                ("decode_kv_bytes", C.c_double), ("decode_flops", C.c_double),
                ("prefill_flops", C.c_double), ("prefill_bytes", C.c_double), ("score_busy_us", C.c_double)]


class Latency(C.Structure):
    _fields_ = [("decode_per_token", C.c_int64), ("prefill_per_token", C.c_int64),
                ("reward_residual", C.c_int64), ("chunk_switch_cost", C.c_int64),
                ("transfer_per_chunk", C.c_int64), ("placement", C.c_int32),
                ("count_prompt_in_prefill", C.c_int32)]


class LengthDist(C.Structure):
    _fields_ = [("kind", C.c_int32), ("fast_len", C.c_int32), ("slow_len", C.c_int32),
                ("cap", C.c_int32), ("p_slow", C.c_double), ("mu_log", C.c_double),
                ("sigma_log", C.c_double), ("table_n", C.c_int32), ("_pad", C.c_int32),
                ("table_len", C.c_int32 * MAX_TABLE), ("table_w", C.c_double * MAX_TABLE)]


class PpoHparams(C.Structure):
    _fields_ = [("gamma", C.c_double), ("lambda_", C.c_double), ("clip_epsilon", C.c_double),
                ("learning_rate", C.c_double), ("value_learning_rate", C.c_double),
                ("kl_coef", C.c_double), ("whiten", C.c_int32), ("value_target", C.c_int32)]


VALUE_MC_RETURN, VALUE_GAE_RETURN = 0, 1


class RunConfig(C.Structure):
    _fields_ = [("mode", C.c_int32), ("steps", C.c_int32), ("batch_size", C.c_int32),
                ("prompt_len", C.c_int32), ("prompt_count", C.c_int64),
                ("delta_init", C.c_int32), ("delta_min", C.c_int32), ("delta_max", C.c_int32),
                ("controller", C.c_int32), ("window", C.c_int32), ("delta_inc", C.c_int32),
                ("delta_dec", C.c_int32), ("chunk_size", C.c_int32),
                ("schedule_mode", C.c_int32), ("tune_chunks", C.c_int32),
                ("n_candidates", C.c_int32), ("chunk_candidates", C.c_int32 * MAX_CANDIDATES),
                ("retune_period", C.c_int32), ("vocab", C.c_int32), ("target_token", C.c_int32),
                ("reward_scale", C.c_double), ("reward_bias", C.c_double),
                ("proxy_kind", C.c_int32), ("proxy_ramp_steps", C.c_int32),
                ("proxy_value", C.c_double), ("proxy_ramp_scale", C.c_double),
                ("fail_after_step", C.c_int32), ("carry_granularity", C.c_int32),
                ("latency", Latency), ("lengths", LengthDist), ("ppo", PpoHparams)]


class StepRecord(C.Structure):
    _fields_ = [("step", C.c_int32), ("finished", C.c_int32), ("wall_ticks", C.c_int64),
                ("deferred", C.c_int32), ("delta", C.c_int32),
                ("has_controller_stat", C.c_int32), ("max_deferrals", C.c_int32),
                ("controller_stat", C.c_double), ("mean_reward", C.c_double),
                ("util_generation", C.c_double), ("util_scoring", C.c_double),
                ("chunk_size", C.c_int32), ("pre_scored", C.c_int32),
                ("step_us", C.c_double), ("update_us", C.c_double), ("ppo_loss", C.c_double),
                ("kl_mean", C.c_double), ("batch_tokens", C.c_int64)]


class ModelDims(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("d_ff", C.c_int32),
                ("vocab", C.c_int32), ("tied", C.c_int32)]


class EngineCfg(C.Structure):
    _fields_ = [("actor", ModelDims), ("reward", ModelDims), ("critic", ModelDims),
                ("ref", ModelDims), ("dtype", C.c_int32), ("device", C.c_int32),
                ("weight_seed", C.c_uint64), ("sample_seed", C.c_uint64),
                ("max_slots", C.c_int32), ("max_prompt_len", C.c_int32),
                ("max_response_len", C.c_int32), ("page_size", C.c_int32),
                ("kv_pages", C.c_int32), ("carry_granularity", C.c_int32),
                ("rank", C.c_int32), ("world", C.c_int32), ("use_graphs", C.c_int32),
                ("train_heads", C.c_int32), ("scorer_sms", C.c_int32), ("nccl_comm", C.c_void_p),
                ("allreduce", C.c_void_p), ("allreduce_ctx", C.c_void_p)]


class PpoStats(C.Structure):
    _fields_ = [("mean_reward", C.c_double), ("ppo_objective", C.c_double),
                ("value_loss", C.c_double), ("kl_mean", C.c_double), ("adv_mean", C.c_double),
                ("adv_std", C.c_double), ("n_tokens", C.c_int64), ("n_samples", C.c_int64),
                ("update_us", C.c_double)]


def struct_sizes():
    return {n: C.sizeof(t) for n, t in [
        ("seq_state", SeqState), ("chunk_task", ChunkTask), ("seq_outcome", SeqOutcome),
        ("ledger", Ledger), ("latency", Latency), ("length_dist", LengthDist),
        ("ppo_hparams", PpoHparams), ("run_config", RunConfig), ("step_record", StepRecord),
        ("model_dims", ModelDims), ("engine_cfg", EngineCfg), ("ppo_stats", PpoStats)]}


# host callbacks of the step loop (include/oppo/oppo.h)
PROMPT_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int64, C.c_int32, C.POINTER(C.c_int32))
STEP_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(StepRecord))
HOST_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.POINTER(C.c_double), C.c_int32)
BATCH_REWARD_FN = C.CFUNCTYPE(C.c_double, C.c_void_p, C.POINTER(C.c_int64), C.c_int32)


class LoopHooks(C.Structure):
    _fields_ = [("prompt", C.c_void_p), ("prompt_ctx", C.c_void_p), ("on_step", C.c_void_p),
                ("step_ctx", C.c_void_p), ("ledgers", C.POINTER(Ledger))]
