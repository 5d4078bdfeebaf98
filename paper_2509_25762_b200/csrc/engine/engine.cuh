// engine.cuh — device state of the OPPO step executor (one per GPU).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "host/sched.hpp"
#include "kernels/gemm.cuh"
#include "kernels/gemm_dec.cuh"
#include "engine/launch.cuh"
#include "kernels/model.cuh"
#include "kernels/attn_mma.cuh"
#include "kernels/attn_dec.cuh"
#include "oppo/oppo.h"

namespace oppo {

enum ModelId { ACTOR = 0, REWARD = 1, CRITIC = 2, REF = 3, N_MODELS = 4 };

struct LayerW {
    void* wqkv;   // [(H+2KV)hd, d]
    float* bqkv;  // [(H+2KV)hd]
    void* wo;     // [d, H hd]
    void* wgu;    // [2 dff, d], rows interleaved (gate_i, up_i)
    void* wdown;  // [d, dff]
    float* ln1;
    float* ln2;
};

struct Model {
    oppo_model_dims dims{};
    bool used = false;
    void* embed = nullptr;    // [V, d] (T)
    void* lm_head = nullptr;  // == embed when tied
    float* lm_master = nullptr;  // fp32 master of lm_head (actor, when training)
    std::vector<LayerW> layers;
    float* final_norm = nullptr;
    float* head = nullptr;    // value / reward head [d] (critic / reward)
    void* k_pool = nullptr;
    void* v_pool = nullptr;
    int64_t layer_stride = 0;  // elements per layer in a pool
    KvView kv(const int32_t* page_table, int max_pages, int page_size) const {
        return KvView{k_pool, v_pool, layer_stride, page_size, dims.n_kv_heads, dims.head_dim,
                      page_table, max_pages};
    }
    int qkv_width() const { return (dims.n_heads + 2 * dims.n_kv_heads) * dims.head_dim; }
    int q_width() const { return dims.n_heads * dims.head_dim; }
};

// Activation workspace of one stream (actor decode or scorer prefill).
struct Work {
    int max_rows = 0;
    int sms = 148;  // SMs of the partition this workspace's stream runs on (grid sizing)
    RowMeta meta{};
    float* x = nullptr;      // residual [R, dmax] fp32
    void* h = nullptr;       // normed   [R, dmax]
    void* qkv = nullptr;     // [R, qkv_max]
    void* q = nullptr;       // [R, qmax]
    void* attn = nullptr;    // [R, qmax]
    void* ff = nullptr;      // [R, dff_max]
    float* head_out = nullptr;   // [R]
    float4* partials = nullptr;  // [R, vocab/128]
    float* tgt_logit = nullptr;  // [R]
    float* lse = nullptr;        // [R]
    void* lm_in = nullptr;       // [R, dmax] gathered lm_head rows
    int32_t* lm_tgt = nullptr;   // [R]
    int32_t* lm_slot = nullptr;
    int32_t* lm_t = nullptr;
    float* gemm_ws = nullptr;    // split-K partials
    size_t gemm_ws_floats = 0;
    int* gemm_cnt = nullptr;     // per-tile arrival counters (zeroed)
    int gemm_cnt_n = 0;
    float* attn_ws_o = nullptr;
    float* attn_ws_ml = nullptr;
    size_t attn_ws_rows = 0;     // rows*heads*splits capacity
    // per-wave metadata staging (device)
    QBlock* qblocks = nullptr;
    Segment* segs = nullptr;
    LmRow* lmrows = nullptr;
    int32_t* pend_src = nullptr;
    int32_t* pend_slot = nullptr;
    int meta_cap = 0;
};

struct TmaKey {
    const void* ptr;
    int rows, cols, box_rows, ld;
    bool operator<(const TmaKey& o) const {
        return std::tie(ptr, rows, cols, box_rows, ld) <
               std::tie(o.ptr, o.rows, o.cols, o.box_rows, o.ld);
    }
};

struct SlotInfo {
    int64_t id = -1;
    int prompt_len = 0;
    int target_len = 0;
    bool ref_pending = false;  // reference lm_head row waiting for its target token
    bool scored_prompt = false;
    std::vector<int> pages;
};

struct Engine {
    oppo_engine_cfg cfg{};
    std::string error;
    int dtype = OPPO_DTYPE_BF16;
    size_t esz = 2;
    int num_sms = 148;
    int sms_actor = 148, sms_scorer = 148;  // fixed SM partition (green contexts) or the whole GPU
    CUgreenCtx gctx_actor = nullptr, gctx_scorer = nullptr;
    Model models[N_MODELS];

    int S = 0, Pmax = 0, Lmax = 0, page_size = 64, max_pages = 0, n_pages = 0;
    int tok_stride = 0;  // Lmax + 2
    std::vector<int> free_slots;
    std::vector<int> free_pages;
    std::unordered_map<int64_t, int> slot_of;
    std::vector<SlotInfo> slots;

    int32_t* d_page_table = nullptr;   // [S, max_pages]
    int32_t* d_prompt = nullptr;       // [S, Pmax]
    int32_t* d_tok = nullptr;          // [S, tok_stride] response tokens, index 1..L
    float* d_old_lp = nullptr;         // [S, tok_stride]
    float* d_ref_lp = nullptr;         // [S, tok_stride]
    float* d_values = nullptr;         // [S, tok_stride] index 1..L (+ L+1 terminal)
    float* d_reward = nullptr;         // [S]
    int32_t* d_target_len = nullptr;   // [S]
    void* d_hf_actor = nullptr;        // [S, tok_stride, d_actor]
    void* d_hf_critic = nullptr;       // [S, tok_stride, d_critic]
    void* d_ref_pending = nullptr;     // [S, d_ref]

    Work wa, ws;                        // actor decode / scorer prefill
    Work wa2;                           // second decode branch (split iterations), rows view into wa.meta
    // concurrent scorer models: critic and reference passes on their own
    // streams (scorer SMs) and workspaces, reading the reward pass's row metadata
    int scorer_streams = 1;
    Work ws_m[2];
    cudaStream_t ss_m[2] = {nullptr, nullptr};
    cudaEvent_t ev_seg = nullptr, ev_m[2] = {nullptr, nullptr};
    cudaEvent_t ev_admit = nullptr;  // end of an admission's writes on su
    // Policy log-probs (and log-sum-exp) of the sampled tokens of every sequence
    // that finished in the last step, computed on the actor SMs while the
    // scorers finish their last wave; oppo_ppo_update reuses them when the
    // lm_head has not changed since (pre_version == lm_version).
    bool pre_lp = false;
    bool prompt_t0 = true;  // streamed: fresh prompts scored in the tick-0 wave (OPPO_PROMPT_T0)
    int64_t lm_version = 0, pre_version = -1;
    std::unordered_map<int64_t, std::pair<int, int>> pre_index;  // seq id -> (token offset, tokens)
    size_t pre_cap = 0;                 // tokens
    void* pre_hf = nullptr;             // [pre_cap, d_actor] gathered final hidden states
    int32_t* pre_tok = nullptr;         // [pre_cap] sampled tokens (targets)
    float* pre_new = nullptr;           // [pre_cap] log pi(token)
    float* pre_lse = nullptr;           // [pre_cap]
    int32_t* pre_meta = nullptr;        // slots + offsets of the gather
    int pre_meta_cap = 0;
    float4* pre_partials = nullptr;     // [pre_chunk, vocab/256]
    float* pre_tgt = nullptr;           // [pre_chunk]
    int pre_chunk = 0;
    cudaEvent_t ev_pre = nullptr;
    cudaStream_t sa2 = nullptr;         // second decode branch stream (actor SMs)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    int dec_split_min = 0;              // decode iterations of >= this many rows run as two concurrent halves
    int prefill_rows = 8192;
    int qblock = 32;  // queries per prefill attention block (bf16: rows = queries x G <= 64)
    cudaStream_t sa = nullptr, ss = nullptr;
    cudaStream_t su = nullptr;  // admission prefill + PPO update: whole GPU (== sa without a partition)
    std::vector<cudaEvent_t> ev_pool;
    std::vector<cudaEvent_t> ev_wave;  // timing events around each scorer wave (start, end): partition busy time
    // K13 chunk hand-off on the device: after the decode iteration that
    // completes a wave's chunks the actor stream publishes the wave's sequence
    // number into a ring of per-chunk ready flags (release store); the scorer
    // stream's first kernel of the wave polls its flag (acquire loads).  Only
    // with eager module loading: under lazy loading the first launch of a
    // kernel waits for the device, so a scorer kernel polling for a flag whose
    // writer (or any kernel ahead of it) is not loaded yet deadlocks -- measured
    // on B200 (tools/probe/flag_probe.cu); per-wave events otherwise.
    static constexpr int kReadyRing = 256;
    uint32_t* d_ready = nullptr;  // [kReadyRing] flags (monotone sequence numbers)
    uint32_t ready_seq = 0;       // last sequence number issued
    bool chunk_flags = false;
    cudaEvent_t ev_begin = nullptr, ev_dec_end = nullptr, ev_sc_end = nullptr, ev_done = nullptr,
                ev_loop0 = nullptr;
    bool step_open = false;
    std::atomic<int64_t> launches{0};  // driver thread and the scorer enqueue thread
    bool pdl = false;  // programmatic dependent launch on the decode / prefill chains
    // decode-path tuning (defaults measured on B200; OPPO_* env overrides for sweeps)
    bool attn_cluster = true;  // split-KV merge in DSMEM (else workspace + combine kernel)
    int attn_per_sm = 4;       // target decode attention CTAs per SM
    int attn_max_split = 0;    // decode split-KV cluster size cap (0: default 8, 1: off)
    int attn_split_minpos = 512;  // fewest context positions per split of a row
    int attn_long_ctx = 768;      // iterations whose longest context reaches this use split-KV attention
    bool attn_long = false;       // set while a long-context decode iteration is enqueued / captured
    int debug_skip = 0;
    bool attn_fused = true;
    int attn_warps = 0;        // decode attention warps per CTA (0 auto, 4 or 8)
    int attn_tp16 = -1;         // 4-warp decode attention with 16-position tiles (hd 64): -1 auto, 0 off, 1 on
    bool rope_epi = true;       // prefill: RoPE + KV append in the q|k|v GEMM epilogue
    int attn_w8_tenths = 20;   // auto rule: 8 warps while CTAs <= tenths/10 x SMs
    int lmhead_dec_max = 32;   // decode lm_head through lmhead_dec.cuh up to this batch (0: off)
    int dec_qkv_max = 96;      // largest batch for which qkv uses the swap-AB decode GEMM
    int dec_gu_max = 64;       // ... gate|up
    int dec_res_max = 192;     // ... O and down (down always: K >= 2048)

    std::map<TmaKey, CUtensorMap> tma_cache;
    std::mutex tma_mu;  // guards tma_cache (decode and scorer launches come from two threads)

    // decode iteration as CUDA graphs, one per active batch size M (kernel
    // arguments depend on M only; the iteration index lives in d_iter)
    DecodeSeq* d_dseq = nullptr;   // [S] fixed, so captured graphs stay valid
    int32_t* d_iter = nullptr;
    std::unordered_map<int, cudaGraphExec_t> decode_graphs;
    std::unordered_map<int, int64_t> decode_graph_launches;

    // PPO update buffers (grown on demand)
    size_t ppo_cap_tok = 0;
    void* ppo_buf = nullptr;
    size_t ppo_buf_bytes = 0;
    void* g_buf = nullptr;   // softmax-grad G [V, chunk]
    void* ht_buf = nullptr;  // transposed hidden [d, chunk]
    int g_chunk = 16384;  // update token chunk (OPPO_G_CHUNK): 4096 -> 16384 cut the update 59.7 -> 55.6 ms
    float* vgrad = nullptr;
    float* g_lm = nullptr;   // DP: lm_head gradient buffer (allreduced)
    void* nccl = nullptr;
    void* train_state = nullptr;  // full-parameter update state (train.cu)
};

// One PPO batch for the full-parameter update (train.cu): the sequences in
// batch order and their per-response-token device arrays.
struct TrainBatch {
    std::vector<int> slot, P, L, off;  // off: response-token prefix sums (n + 1)
    int rows_max = 16384;              // training rows per micro-batch (whole sequences)
    const int32_t* tok = nullptr;      // [N] sampled tokens
    float* adv = nullptr;              // [N] GAE advantages (whitened in place by ppo_clip)
    const float* old_lp = nullptr;     // [N]
    const float* ret = nullptr;        // [N] critic targets
    float* new_lp = nullptr;           // [N] out: current-policy log-probs
    float* lse = nullptr;              // [N] out
    float* dobj = nullptr;             // [N] out: dObj/dlogp
    const double* stats = nullptr;     // whitening moments (sum, sumsq, n) or null
    float clip_eps = 0.2f, inv_n = 1.f;
    double* part = nullptr;            // >= 1024 doubles
    double* obj_acc = nullptr;         // += sum of clipped-objective terms
    float* sq = nullptr;               // [N] out: squared value errors
    float* v_new = nullptr;            // [N] out (optional): current critic values
    void* meta_dev = nullptr;          // device staging of the micro-batch metadata
    size_t meta_cap = 0;
};

// engine.cu
Engine* engine_new(const oppo_engine_cfg& cfg);
void engine_free(Engine* e);

// train.cu
template <class T>
void train_full(Engine& e, TrainBatch& b, const oppo_ppo_hparams& hp, bool dp, cudaStream_t st);
void train_free(Engine& e);
std::vector<std::pair<void*, size_t>> train_tensors(Engine& e, cudaStream_t st);
const float* train_master(Engine& e, int model, const std::string& name, int layer);
// engine.cu
void dp_allreduce_pub(Engine& e, void* buf, int64_t count, bool f64, cudaStream_t st);
void dp_allreduce_bucket(Engine& e, const std::vector<std::pair<float*, int64_t>>& bufs, cudaStream_t st);

// gemm_host.cu
void gemm_run(Engine& e, Work& w, cudaStream_t st, const void* x, int M, int K, int ldx,
              const void* wt, int N, int ldw, const EpiParams& ep);
void gemm_standalone(int dtype, int M, int N, int K, const void* x, const void* w,
                     const float* bias, void* y, int epi, cudaStream_t st);
// Y[M,N] = A . B^T with either operand MN-major (stored transposed, a: [K][M]
// ld lda, b: [K][N] ld ldb) -- the update's wgrad / dgrad GEMMs read dY, X
// and W in place instead of transposed copies.
void gemm_run_t(Engine& e, Work& w, cudaStream_t st, const void* a, int a_mn, int lda, const void* b, int b_mn,
                int ldb, int M, int N, int K, const EpiParams& ep);
void gemm_standalone_t(int dtype, int M, int N, int K, const void* a, int a_mn, int lda, const void* b, int b_mn,
                       int ldb, void* y, int epi, cudaStream_t st);
int gemm_dec_run(Engine& e, Work& w, cudaStream_t st, const void* x, int M, int K, int ldx,
                 const void* wt, int N, int ldw, int mode, void* y, int ldy, const float* bias);
int gemm_dec_impl(Engine* e, cudaStream_t st, const void* x, int M, int K, int ldx, const void* wt,
                  int N, int ldw, int mode, void* y, int ldy, const float* bias, float* ws,
                  size_t ws_floats, int num_sms, bool pdl);
const CUtensorMap& cached_map_pub(Engine* e, const void* ptr, int rows, int cols, int ld, int box_rows,
                                  CUtensorMap& scratch);
void lmhead_dec_run(Engine& e, Work& w, cudaStream_t st, const void* x, int M, int K, const void* wt,
                    int V, float4* partials, const uint64_t* keys);
CUtensorMap make_tma_2d(const void* ptr, int rows, int cols, int ld, int box_rows);
int gemm_logit_tiles(int dtype, int N);  // partial tiles per row of an EPI_LOGITS GEMM
void gemm_with_params(int dtype, int M, int N, int K, const void* x, const void* w,
                      const EpiParams& ep, cudaStream_t st);

}  // namespace oppo
