/*
 * oppo.h — C ABI of the B200-native OPPO PPO-RLHF step (liboppo.so).
 *
 * This is the drop-in boundary for the reference's generation-plus-scoring hot
 * path.  The reference (`/root/reference/proj/core`, C++20, namespace rlpipe)
 * exposes that path only as a C++ API over value types; every entry point
 * below names the reference interface it replaces (file:line under
 * /root/reference).  Conventions kept from the reference:
 *
 *   - errors: every call returns oppo_status.  ConfigError (errors.hpp:9-12)
 *     -> OPPO_ERR_CONFIG, InputError (errors.hpp:15-18) -> OPPO_ERR_INPUT,
 *     InternalError (errors.hpp:21-24) -> OPPO_ERR_INTERNAL; GPU-side failures
 *     add OPPO_ERR_CUDA / OPPO_ERR_NCCL.  The message of the last failure is
 *     returned by oppo_last_error() (thread-local for engine-free calls, per
 *     engine for engine calls) so a C++ shim can rethrow the same types.
 *   - purity/ownership: functions that are pure in the reference (run_step,
 *     engine.hpp:90) only read their inputs; functions that mutate in the
 *     reference (refill/select_finished, overcommit.hpp:48,61) take in/out
 *     arrays.  Host arrays are caller-owned; device memory is engine-owned.
 *   - threading: one driver thread per engine.
 *
 * No torch types appear here: plain pointers and sizes only.
 */
#ifndef OPPO_OPPO_H
#define OPPO_OPPO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t oppo_status;
enum {
    OPPO_OK = 0,
    OPPO_ERR_CONFIG = 1,   /* rlpipe::ConfigError   */
    OPPO_ERR_INPUT = 2,    /* rlpipe::InputError    */
    OPPO_ERR_INTERNAL = 3, /* rlpipe::InternalError */
    OPPO_ERR_CUDA = 4,
    OPPO_ERR_NCCL = 5,
};

/* ------------------------------------------------------------------ values */

/* rlpipe::SequenceState + PromptRequest (model.hpp:23-36, :12-16). */
typedef struct oppo_seq_state {
    int64_t id;
    int32_t prompt_len;
    int32_t arrival_step;
    int32_t target_len;       /* full response length, drawn at admission */
    int32_t generated;        /* decoded tokens kept so far                */
    int32_t prefilled_tokens; /* response tokens prefilled downstream      */
    int32_t chunks_emitted;
    int32_t chunks_prefilled;
    int32_t finished;
    int32_t scored;
    int32_t admitted_at;
    int32_t deferrals;
    int32_t _pad;
} oppo_seq_state;

/* rlpipe::ChunkTask (chunking.hpp:23-27), flattened with its sequence id. */
typedef struct oppo_chunk_task {
    int64_t seq_id;
    int32_t first;
    int32_t last;
    int32_t index;
    int32_t needs_decode;
} oppo_chunk_task;

/* rlpipe::SequenceOutcome minus the per-chunk tick vectors (engine.hpp:59-69). */
typedef struct oppo_seq_outcome {
    int64_t seq_id;
    int64_t score_ready; /* tick, or -1 when not scored within the step */
    int32_t tokens_decoded;
    int32_t tokens_prefilled;
    int32_t decode_chunks_completed;
    int32_t prefill_tasks_completed;
    int32_t carry_prefill_completed;
    int32_t _pad;
} oppo_seq_outcome;

/* rlpipe::ResourceLedger (engine.hpp:77-83) plus measured device time. */
typedef struct oppo_ledger {
    int64_t wall;
    int64_t busy_generation;
    int64_t busy_scoring;
    int64_t work_generation;
    int64_t work_scoring;
    /* measured on the GPU (CUDA events); 0 for logical-only calls */
    double step_us;        /* whole step: decode + scorer waves + drain   */
    double decode_us;      /* actor stream busy time                      */
    double score_us;       /* scorer stream busy time                     */
    int64_t decode_iters;  /* lockstep decode iterations executed         */
    int64_t decode_tokens; /* tokens sampled (including discarded tails)  */
    int64_t prefill_tokens;/* scorer tokens prefilled (per scorer)        */
    int64_t kernel_launches;
    /* actor decode loop alone (first decode iteration .. last), and its
     * algorithmic HBM bytes: actor weights (non-embedding + lm_head) once per
     * iteration + the KV cache each active row reads and appends */
    double decode_loop_us;
    double decode_weight_bytes;
    double decode_kv_bytes;
    /* algorithmic work of the step: decode flops (2 P_dec + 4 L H hd ctx
     * per sampled token), scorer prefill flops (linear layers, causal attention and
     * the reference model's lm_head rows) and bytes (each pass's weights of the
     * three scorers + the KV they append and read) */
    double decode_flops;
    double prefill_flops;
    double prefill_bytes;
    /* measured busy time of the scorer partition: the sum over the step's
     * waves of (wave end - wave start) on the scorer stream (engine.cpp:225-233's
     * busy_scoring, in us); the actor partition's is decode_loop_us */
    double score_busy_us;
} oppo_ledger;

enum { OPPO_MODE_STREAMED = 0, OPPO_MODE_SEQUENTIAL = 1 };      /* ScheduleMode */
enum { OPPO_PLACE_COLOCATED = 0, OPPO_PLACE_DISAGGREGATED = 1 }; /* Placement    */
enum { OPPO_LEN_TWO_POINT = 0, OPPO_LEN_LOGNORMAL = 1, OPPO_LEN_EMPIRICAL = 2 };
enum { OPPO_DELTA_FIXED = 0, OPPO_DELTA_ALG1 = 1, OPPO_DELTA_EQ4 = 2 };   /* DeltaMode */
enum { OPPO_RUN_SIMULATE = 0, OPPO_RUN_TRAIN = 1, OPPO_RUN_TUNE = 2 };  /* RunMode   */
enum { OPPO_CARRY_CHUNK = 0, OPPO_CARRY_TOKEN = 1 };

/* rlpipe::LatencyModel (model.hpp:43-53). */
typedef struct oppo_latency {
    int64_t decode_per_token;
    int64_t prefill_per_token;
    int64_t reward_residual;
    int64_t chunk_switch_cost;
    int64_t transfer_per_chunk;
    int32_t placement;
    int32_t count_prompt_in_prefill;
} oppo_latency;

#define OPPO_MAX_TABLE 64
/* rlpipe::LengthDistribution (model.hpp:65-84). */
typedef struct oppo_length_dist {
    int32_t kind;
    int32_t fast_len;
    int32_t slow_len;
    int32_t cap;
    double p_slow;
    double mu_log;
    double sigma_log;
    int32_t table_n;
    int32_t _pad;
    int32_t table_len[OPPO_MAX_TABLE];
    double table_w[OPPO_MAX_TABLE];
} oppo_length_dist;

/* rlpipe::PpoHyperparams (ppo.hpp:12-20) plus the GPU-only KL/whitening knobs. */
typedef struct oppo_ppo_hparams {
    double gamma;
    double lambda;
    double clip_epsilon;
    double learning_rate;
    double value_learning_rate;
    double kl_coef;      /* 0 -> terminal reward only, as the reference */
    int32_t whiten;      /* 0 -> raw GAE advantages, as the reference    */
    int32_t value_target; /* critic regression target: OPPO_VALUE_MC_RETURN (0): gamma-discounted
                             return of the terminal reward, as the reference's value fit
                             (ppo.cpp:296-314); OPPO_VALUE_GAE_RETURN (1): GAE lambda-return
                             adv + V of the KL-shaped rewards (TRL style) */
} oppo_ppo_hparams;
#define OPPO_VALUE_MC_RETURN 0
#define OPPO_VALUE_GAE_RETURN 1

#define OPPO_MAX_CANDIDATES 16
/* rlpipe::RunConfig (config.hpp:28-77), the fields the hot path reads. */
typedef struct oppo_run_config {
    int32_t mode;
    int32_t steps;
    int32_t batch_size;
    int32_t prompt_len;
    int64_t prompt_count; /* -1 unbounded */
    int32_t delta_init;
    int32_t delta_min;
    int32_t delta_max;
    int32_t controller;
    int32_t window;
    int32_t delta_inc;
    int32_t delta_dec;
    int32_t chunk_size;
    int32_t schedule_mode;
    int32_t tune_chunks;
    int32_t n_candidates;
    int32_t chunk_candidates[OPPO_MAX_CANDIDATES];
    int32_t retune_period;
    int32_t vocab;        /* toy env only (ppo.hpp:55-62) */
    int32_t target_token;
    double reward_scale;
    double reward_bias;
    int32_t proxy_kind;   /* RewardProxy (config.hpp:20-26) */
    int32_t proxy_ramp_steps;
    double proxy_value;
    double proxy_ramp_scale;
    int32_t fail_after_step;
    int32_t carry_granularity; /* GPU extension: chunk (reference) | token */
    oppo_latency latency;
    oppo_length_dist lengths;
    oppo_ppo_hparams ppo;
} oppo_run_config;

/* rlpipe::StepRecord (driver.hpp:13-24) plus measured GPU time. */
typedef struct oppo_step_record {
    int32_t step;
    int32_t finished;
    int64_t wall_ticks;
    int32_t deferred;
    int32_t delta;
    int32_t has_controller_stat;
    int32_t max_deferrals;
    double controller_stat;
    double mean_reward;
    double util_generation;
    double util_scoring;
    int32_t chunk_size;
    int32_t pre_scored;
    double step_us;     /* generation + scoring (reference definition, driver.cpp:173) */
    double update_us;   /* PPO update (K8-K12)                                          */
    double ppo_loss;
    double kl_mean;
    int64_t batch_tokens;
} oppo_step_record;

/* Per-step callback of the step loop (run after selection, update and the
 * controller step of each step); a non-zero return ends the loop. */
typedef int32_t (*oppo_step_fn)(void* ctx, const oppo_step_record* rec);

/* ------------------------------------------------ host scheduler (no GPU) */

/* Defaults identical to RunConfig{} (config.hpp:28-77). */
void oppo_run_config_default(oppo_run_config* cfg);
/* RunConfig::baseline (config.cpp:411-420): delta 0, Fixed, Sequential, no tuner. */
void oppo_run_config_baseline(const oppo_run_config* cfg, oppo_run_config* out);
/* RunConfig::validate (config.cpp:253-289). */
oppo_status oppo_run_config_validate(const oppo_run_config* cfg);

/* Rng::derive(seed, purpose) then n draws (rng.hpp:20-54). kind 0 u64, 1 uniform01, 2 normal. */
oppo_status oppo_rng_draws(uint64_t seed, const char* purpose, int32_t kind, int64_t n,
                           void* out);
/* sample_response_length (model.cpp:50-72) n times on Rng::derive(seed, "lengths"). */
oppo_status oppo_sample_lengths(const oppo_length_dist* dist, uint64_t seed, int64_t n,
                                int32_t* out);

/* build_schedule (chunking.cpp:20-48).  tasks has room for cap entries;
 * *n_tasks receives the count (tasks grouped per sequence, in input order). */
oppo_status oppo_build_schedule(const oppo_seq_state* seqs, int32_t n, int32_t chunk_size,
                                int32_t mode, oppo_chunk_task* tasks, int32_t cap,
                                int32_t* n_tasks);

/* run_step (engine.cpp:24-223) on the logical clock of the GPU executor: the
 * lockstep model {decode=1, prefill=0, residual=0, disaggregated}.  This is the
 * decision function the GPU executor obeys; carry_granularity=token credits
 * decoded-but-unfinished chunk tails (north_star extension of engine.cpp:190). */
oppo_status oppo_plan_step(const oppo_seq_state* active, int32_t n, int32_t chunk_size,
                           int32_t mode, int32_t stop_after, int32_t carry_granularity,
                           oppo_seq_outcome* out, oppo_ledger* ledger);

/* select_finished (overcommit.cpp:30-95); entries in/out (n in, *n_out out). */
oppo_status oppo_select_finished(oppo_seq_state* entries, int32_t n,
                                 const oppo_seq_outcome* outcomes, int32_t n_out_in,
                                 int32_t batch_size, oppo_seq_state* batch, int32_t* n_batch,
                                 int32_t* n_remaining, int32_t* short_batch);

/* DeltaController::update (overcommit.cpp:134-155).  history in/out. */
oppo_status oppo_delta_update(int32_t mode, int32_t window, int32_t dmin, int32_t dmax,
                              int32_t inc, int32_t dec, double* history, int32_t* n_hist,
                              int32_t delta, int32_t* new_delta, int32_t* has_stat,
                              double* stat);

/* make_tuner + retune_chunk_size replay (chunking.cpp:61-100): folds
 * (candidate, measurement) pairs in order; chosen[i] = current after pair i. */
oppo_status oppo_tuner_replay(const int32_t* candidates, int32_t n_cand, int32_t window,
                              const int32_t* meas_cand, const double* meas, int32_t n_meas,
                              int32_t* chosen);

/* sizeof of every struct above, in declaration order (binding layout check). */
int32_t oppo_abi_sizes(int64_t* out, int32_t cap);

/* Scheduler-only run of the step loop (driver.cpp:103-195) with the logical
 * executor; no GPU.  Records one oppo_step_record per step and, if sel_ids is
 * non-NULL, the selected ids of each step (batch_size slots per step, -1 pad). */
/* The logical loop as rank `rank` of `world` (CPU; the data-parallel
 * decisions without a GPU): sums go through `allreduce` (in place, n doubles),
 * and in simulate mode the controller's reward is batch_reward(selected ids)
 * when given (else the reference's proxy). */
typedef int32_t (*oppo_host_allreduce_fn)(void* ctx, double* v, int32_t n);
typedef double (*oppo_batch_reward_fn)(void* ctx, const int64_t* ids, int32_t n);
oppo_status oppo_run_seed_logical_dp(const oppo_run_config* cfg, uint64_t seed, int32_t rank, int32_t world,
                                     oppo_host_allreduce_fn allreduce, void* allreduce_ctx,
                                     oppo_batch_reward_fn batch_reward, void* reward_ctx,
                                     oppo_step_record* records, int32_t* n_records, int64_t* sel_ids);
oppo_status oppo_run_seed_logical(const oppo_run_config* cfg, uint64_t seed,
                                  oppo_step_record* records, int32_t* n_records,
                                  int64_t* sel_ids);

const char* oppo_last_error_global(void);

/* ------------------------------------------------------------- GPU engine */

typedef struct oppo_model_dims {
    int32_t n_layers;
    int32_t d_model;
    int32_t n_heads;
    int32_t n_kv_heads;
    int32_t head_dim;
    int32_t d_ff;
    int32_t vocab;
    int32_t tied; /* lm_head shares the embedding */
} oppo_model_dims;

enum { OPPO_DTYPE_F32 = 0, OPPO_DTYPE_BF16 = 1 };

/* Host-provided sum-allreduce used instead of NCCL when nccl_comm is NULL and
 * world > 1 (e.g. a gloo process group in tests, or another transport):
 * reduce `count` elements (dtype 0 f32, 1 f64) of the DEVICE buffer in place
 * across ranks; work already enqueued on `stream` must be visible first.
 * Returns 0 on success. */
typedef int32_t (*oppo_allreduce_fn)(void* ctx, void* device_buf, int64_t count, int32_t dtype,
                                     void* stream);

typedef struct oppo_engine_cfg {
    oppo_model_dims actor;
    oppo_model_dims reward;
    oppo_model_dims critic;
    oppo_model_dims ref;
    int32_t dtype;
    int32_t device;
    uint64_t weight_seed;
    uint64_t sample_seed;
    int32_t max_slots;        /* B + delta_max (+ carried)            */
    int32_t max_prompt_len;
    int32_t max_response_len; /* lengths.cap                          */
    int32_t page_size;        /* KV tokens per page                   */
    int32_t kv_pages;         /* per model; 0 -> enough for all slots */
    int32_t carry_granularity;
    int32_t rank;
    int32_t world;
    int32_t use_graphs;       /* capture the decode iteration in a CUDA graph */
    int32_t train_heads;      /* PPO update: 0 none, 1 lm_head (actor) + value head (critic)
                                 only, 2 every parameter of actor and critic (K11/K12) */
    int32_t scorer_sms;       /* fixed SM partition: SMs for the scorer stream (green
                                 contexts, multiple of 8), the rest run the actor; 0 = shared */
    void* nccl_comm;          /* ncclComm_t or NULL (single GPU)       */
    oppo_allreduce_fn allreduce; /* used when nccl_comm is NULL and world > 1 */
    void* allreduce_ctx;
} oppo_engine_cfg;

typedef struct oppo_engine oppo_engine;

/* Device-side replacement for the rlpipe driver loop state; one per GPU. */
oppo_status oppo_engine_create(const oppo_engine_cfg* cfg, oppo_engine** out);
void oppo_engine_destroy(oppo_engine* e);
const char* oppo_last_error(const oppo_engine* e);

/* Admission side effects of refill (overcommit.cpp:11-28): allocate a slot and
 * the prompt for each new sequence.  prompt tokens: n x prompt_len, or NULL to
 * draw them from the synthetic prompt stream keyed by (sample_seed, id). */
oppo_status oppo_admit(oppo_engine* e, const oppo_seq_state* seqs, int32_t n,
                       const int32_t* prompt_tokens);

/* run_step (engine.hpp:91-93) executed on the GPU: lockstep batched decode of
 * the actor over all active sequences, chunk waves streamed to the reward /
 * critic / reference prefill on a concurrent stream (streamed mode) or scored
 * after generation (sequential mode), cut at the stop_after-th finisher. */
oppo_status oppo_run_step(oppo_engine* e, const oppo_seq_state* active, int32_t n_active,
                          int32_t chunk_size, int32_t mode, int32_t stop_after,
                          oppo_seq_outcome* out, oppo_ledger* ledger);

typedef struct oppo_ppo_stats {
    double mean_reward;
    double ppo_objective; /* clipped surrogate, token mean (ppo.cpp:101-120) */
    double value_loss;
    double kl_mean;
    double adv_mean;
    double adv_std;
    int64_t n_tokens;
    int64_t n_samples;
    double update_us;
} oppo_ppo_stats;

/* fill_values + toy_rlhf_step (ppo.cpp:274-317) for the selected batch. */
oppo_status oppo_ppo_update(oppo_engine* e, const int64_t* batch_ids, int32_t n,
                            const oppo_ppo_hparams* hp, oppo_ppo_stats* out);

/* Free the KV pages / slot of finished sequences. */
oppo_status oppo_release(oppo_engine* e, const int64_t* ids, int32_t n);

/* Engine checkpoint between steps (the reference keeps its
 * carry buffer in memory only, driver.cpp:103-195): slot table, page tables,
 * prompts, tokens / log-probs / values / rewards, cached hidden states, the
 * KV pages of every admitted sequence in all four models, and the trained
 * heads.  Load into a fresh engine created with the same configuration
 * (OPPO_ERR_CONFIG otherwise); the host-side buffer of oppo_seq_state,
 * Delta controller and tuner state stay the caller's (plain data). */
oppo_status oppo_engine_save(oppo_engine* e, const char* path);
oppo_status oppo_engine_load(oppo_engine* e, const char* path);

/* Parity dump of one sequence: tokens, old log-probs, ref log-probs, values (len+1),
 * reward.  cap = room in the token-indexed arrays. */
oppo_status oppo_read_rollout(oppo_engine* e, int64_t id, int32_t* tokens, float* old_lp,
                              float* ref_lp, float* values, float* reward, int32_t cap,
                              int32_t* len);

/* Full OPPO run on the GPU: the driver loop (driver.cpp:103-195) with run_step
 * replaced by oppo_run_step and fill_values/toy_rlhf_step by oppo_ppo_update. */
oppo_status oppo_run_seed(oppo_engine* e, const oppo_run_config* cfg, uint64_t seed,
                          oppo_step_record* records, int32_t* n_records, int64_t* sel_ids);

/* The reference's PromptSource seam (overcommit.hpp:16-20): prompt tokens of
 * sequence `id` (prompt_len of them) into tokens_out; non-zero = failure. */
typedef int32_t (*oppo_prompt_fn)(void* ctx, int64_t id, int32_t prompt_len, int32_t* tokens_out);
typedef struct oppo_loop_hooks {
    oppo_prompt_fn prompt;  /* NULL: synthetic prompt stream keyed by (sample_seed, id) */
    void* prompt_ctx;
    oppo_step_fn on_step;   /* NULL: none */
    void* step_ctx;
    oppo_ledger* ledgers;   /* NULL or [cfg->steps]: each step's ledger */
} oppo_loop_hooks;
/* run_seed with host hooks.  Data parallel when the engine was created with
 * world > 1: rank r serves prompt ids = r (mod world), draws its
 * lengths from Rng::derive(seed ^ r, "lengths"), the Delta controller is fed
 * the global mean reward and the tuner the max step time over the ranks.
 * Refill defers a sequence while the engine lacks a slot or KV pages for it
 * (admission control; the reference's refill never defers). */
oppo_status oppo_run_seed_ex(oppo_engine* e, const oppo_run_config* cfg, uint64_t seed,
                             const oppo_loop_hooks* hooks, oppo_step_record* records, int32_t* n_records,
                             int64_t* sel_ids);

/* Data-parallel plumbing: one NCCL communicator over the GPUs of
 * the box; pass it as oppo_engine_cfg.nccl_comm with rank/world.  The engine
 * then allreduces the whitening / reward statistics and the gradients of the
 * trained tensors inside oppo_ppo_update (full-parameter update: one grouped
 * allreduce per layer on a comm stream, overlapped with the rest of the
 * backward).  Rank 0 creates the id and ships it to
 * the other ranks (e.g. torch.distributed broadcast). */
#define OPPO_NCCL_ID_BYTES 128
oppo_status oppo_nccl_unique_id(uint8_t* out /* OPPO_NCCL_ID_BYTES */);
oppo_status oppo_nccl_comm_create(const uint8_t* id, int32_t world, int32_t rank, int32_t device,
                                  void** comm);
oppo_status oppo_nccl_comm_destroy(void* comm);

/* Prompt tokens of an admitted sequence (synthetic stream or caller-provided). */
oppo_status oppo_read_prompt(oppo_engine* e, int64_t id, int32_t* out, int32_t cap, int32_t* len);

/* Copies one weight tensor as fp32 (oracle parity).  model: 0 actor, 1 reward,
 * 2 critic, 3 ref.  name: embed lm_head final_norm head wqkv bqkv wo wgu
 * wdown ln1 ln2 (layer-indexed for the last seven). */
oppo_status oppo_get_tensor(oppo_engine* e, int32_t model, const char* name, int32_t layer,
                            float* out, int64_t cap, int64_t* n_out);

/* Sets the thread-local message read by oppo_last_error_global(). */
void oppo_set_global_error(const char* msg);

/* --------------------------------------------- kernel-level entry points
 * Device pointers; used by the parity tests to drive one kernel at a time. */

/* K8+K10: per-token GAE (compute_gae, ppo.cpp:71-85, terminal reward
 * ppo.cpp:87-91) + clipped objective (ppo.cpp:101-120) + d objective / d logp
 * (the scalar of clipped_objective_grad, ppo.cpp:138-177) for a ragged batch.
 * fp64 (is_f64=1) or fp32.  offsets: n_seq+1 prefix of token counts; values
 * has len+1 entries per sequence at offsets[i]+i. */
oppo_status oppo_k_ppo_token(int32_t is_f64, int32_t n_seq, const int32_t* d_offsets,
                             const void* d_rewards_seq, const void* d_token_rewards,
                             const void* d_values, const void* d_new_lp,
                             const void* d_old_lp, double gamma, double lambda, double eps,
                             int32_t whiten, void* d_adv, void* d_returns, void* d_dobj_dlp,
                             void* d_obj_sum, void* stream);

/* bf16/f32 GEMM Y[M,N] = X[M,K] . W[N,K]^T (+bias) through the engine's GEMM
 * (tcgen05/TMA for bf16, SIMT for f32).  epilogue 0 store, 1 add to f32 out. */
oppo_status oppo_k_gemm(int32_t dtype, int32_t M, int32_t N, int32_t K, const void* d_x,
                        const void* d_w, const void* d_bias, void* d_y, int32_t epilogue,
                        void* stream);

/* The same GEMM with either operand MN-major (stored transposed: A as
 * d_a[K][M] with leading dimension lda, B as d_b[K][N] with ldb; K-major
 * operands are d_a[M][K] / d_b[N][K]), as the full-parameter update reads dY,
 * X and W in place for its wgrad / dgrad GEMMs.  epilogue 0 store (dtype),
 * 1 add to f32 out, 5 store f32; d_y is [M][N]. */
oppo_status oppo_k_gemm_t(int32_t dtype, int32_t M, int32_t N, int32_t K, const void* d_a, int32_t a_mn,
                          int32_t lda, const void* d_b, int32_t b_mn, int32_t ldb, void* d_y, int32_t epilogue,
                          void* stream);

/* Decode-shaped GEMM (swap-AB tcgen05, M <= 512 tokens) behind the actor's
 * decode iteration.  mode 0: fp32 split-K partials into d_ws[splits][M][N]
 * (*splits receives the count; the sum over splits is Y); mode 1: SwiGLU over
 * interleaved (gate, up) weight rows into d_y[M][N/2] bf16; mode 2: store
 * (+bias) into d_y[M][N] bf16.  K must be a multiple of 64. */
oppo_status oppo_k_gemm_dec(int32_t M, int32_t N, int32_t K, const void* d_x, const void* d_w,
                            const void* d_bias, void* d_y, int32_t mode, void* d_ws,
                            int64_t ws_floats, int32_t* splits, void* stream);

/* Times the engine GEMM alone (epilogue >= 16: the decode GEMM, mode epilogue-16) over `copies` distinct weight matrices; avg_us per launch. */
oppo_status oppo_k_gemm_bench(int32_t M, int32_t N, int32_t K, int32_t copies, int32_t reps,
                              int32_t epilogue, float* avg_us);

#ifdef __cplusplus
}
#endif
#endif /* OPPO_OPPO_H */
