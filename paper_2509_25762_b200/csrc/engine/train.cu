// train.cu — the full-parameter PPO update: actor
// and critic trained through every layer, as the reference's
// toy_rlhf_step updates every policy parameter (ppo.cpp:281-317:
// theta += lr * clipped_objective_grad, value fit toward discounted returns).
//
// Per model, the update's sequences (prompt + response, minus the last
// response token) are packed into micro-batches of whole sequences.  For each
// micro-batch: a training forward that keeps every layer's input residual,
// post-RoPE q|k|v, attention output + log-sum-exp, mid residual and gate|up
// pre-activation; the loss head (actor: lm_head + log-softmax + clipped
// surrogate, dObj/dlogits through the softmax-grad GEMM epilogue; critic:
// value head + squared error to the returns); then the backward, layer by
// layer.  The dgrad GEMMs (dX = dY W) and wgrad GEMMs (dW += dY^T X over the
// token dimension, into fp32 gradient buffers) read W, dY and X in place:
// the tcgen05 GEMM takes either operand MN-major (K-outer storage, TMA boxes of
// [64 k][64 mn], transposed UMMA descriptors), so no transposed copy of a
// weight or activation is ever materialised.  SwiGLU runs in the gate|up
// GEMM's epilogue (forward: product + saved pre-activations; backward: the
// dgrad GEMM of the down projection writes d(gate, up) directly), and the
// RMSNorm backward emits the bf16 copy of the residual gradient the next
// GEMMs read.
// Data-parallel runs allreduce the gradients in per-layer buckets overlapped
// with the backward: in the last micro-batch, as soon as layer
// l's gradients are final, a comm stream waits for them, runs one grouped NCCL
// allreduce of the layer's tensors and applies their SGD step to the fp32
// masters (re-rounding the bf16 compute weights) while the compute stream
// goes on with layers l-1 .. 0; the embedding / lm_head / final norm / head
// form the last bucket.  Without a communicator (or with the host allreduce
// hook) the tensors are reduced and applied after the last micro-batch.
#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <functional>
#include <string>
#include <type_traits>
#include <vector>

#include "engine.cuh"
#include "kernels/ppo.cuh"
#include "kernels/train.cuh"
#include "kernels/attn_train_mma.cuh"

namespace oppo {

namespace {

constexpr float kEps = 1e-6f;
constexpr float kTheta = 1e6f;
constexpr int kColParts = 1024;  // block partial rows of the column sums (ts.colp)

inline int cdiv(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

void* dalloc(size_t bytes) {
    void* p = nullptr;
    OPPO_CUDA_CHECK(cudaMalloc(&p, bytes ? bytes : 16));
    return p;
}

// One trainable tensor of a model.
struct PT {
    void* w = nullptr;        // compute tensor (T matrix or fp32 vector)
    float* master = nullptr;  // fp32 master (bf16 matrices), else null (w is fp32)
    float* grad = nullptr;    // fp32 gradient, same layout as w
    int64_t rows = 0, cols = 1;
    bool matrix = false;
    int64_t n() const { return rows * cols; }
};

struct LayerT {
    PT wqkv, bqkv, wo, wgu, wdown, ln1, ln2;
};

struct ModelT {
    bool ready = false;
    PT embed, lm_head, final_norm, head;  // lm_head.w == embed.w when tied
    std::vector<LayerT> layers;
    std::vector<PT*> all() {
        std::vector<PT*> v{&embed};
        if (lm_head.w && lm_head.w != embed.w) v.push_back(&lm_head);
        v.push_back(&final_norm);
        if (head.w) v.push_back(&head);
        for (auto& L : layers)
            for (PT* p : {&L.wqkv, &L.bqkv, &L.wo, &L.wgu, &L.wdown, &L.ln1, &L.ln2}) v.push_back(p);
        return v;
    }
};

// Scratch of one micro-batch (grown on demand).
struct Scratch {
    size_t cap = 0;
    std::vector<void*> bufs;
    void* take(size_t bytes) {
        void* p = dalloc(bytes);
        bufs.push_back(p);
        return p;
    }
    void release() {
        for (void* p : bufs) cudaFree(p);
        bufs.clear();
        cap = 0;
    }
};

}  // namespace

struct TrainState {
    ModelT m[N_MODELS];
    Scratch scr;
    int rows_cap = 0;  // training rows the scratch is sized for
    // per-layer saved activations: residual inputs (fp32), normed inputs of
    // the attention / MLP blocks, post-RoPE q|k|v, attention output + lse,
    // (gate, up) pre-activations and the SwiGLU product
    std::vector<float*> x_in, x_mid, lse, rstd1, rstd2;
    std::vector<void*> h1, h2, qkv, o, gu, ff;
    // transients
    float* dkv_part = nullptr;  // [G][rows][2 * KV * hd] head-split dK / dV partials
    float *x = nullptr, *dx = nullptr, *dh = nullptr, *dqkv = nullptr, *dvec = nullptr, *gscr = nullptr,
          *colp = nullptr, *head_out = nullptr, *dhf_c = nullptr;
    void *hf = nullptr, *dgu = nullptr, *dxc = nullptr, *dO = nullptr, *dqkvc = nullptr, *hf_resp = nullptr,
         *Gt = nullptr;
    int32_t *tok = nullptr, *pos = nullptr;
    int g_rows = 0;  // lm_head gradient chunk (rows)
    // gradient buckets of data-parallel updates: comm stream + hand-off events
    cudaStream_t comm = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_comm = nullptr;
};

void train_free(Engine& e) {
    auto* ts = static_cast<TrainState*>(e.train_state);
    if (!ts) return;
    ts->scr.release();
    if (ts->comm) cudaStreamDestroy(ts->comm);
    if (ts->ev_ready) cudaEventDestroy(ts->ev_ready);
    if (ts->ev_comm) cudaEventDestroy(ts->ev_comm);
    for (auto& m : ts->m)
        for (PT* p : m.all()) {
            if (p->grad) cudaFree(p->grad);
            // the actor's lm_head master belongs to the engine (freed in engine_free)
            if (p->master && p->master != e.models[ACTOR].lm_master) cudaFree(p->master);
        }
    delete ts;
    e.train_state = nullptr;
}

namespace {

PT make_pt(Engine& e, void* w, int64_t rows, int64_t cols, bool matrix, float* master_existing, cudaStream_t st) {
    PT p;
    p.w = w;
    p.rows = rows;
    p.cols = cols;
    p.matrix = matrix;
    p.grad = static_cast<float*>(dalloc(p.n() * 4));
    if (matrix && e.dtype == OPPO_DTYPE_BF16) {
        if (master_existing) {
            p.master = master_existing;
        } else {
            p.master = static_cast<float*>(dalloc(p.n() * 4));
            convert<__nv_bfloat16, float><<<cdiv(p.n(), 256), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(w),
                                                                             p.master, p.n());
        }
    }
    return p;
}

void setup_model(Engine& e, TrainState& ts, int mid, cudaStream_t st) {
    ModelT& mt = ts.m[mid];
    if (mt.ready) return;
    Model& m = e.models[mid];
    const auto& d = m.dims;
    const int64_t D = d.d_model, V = d.vocab, F = d.d_ff, qkv = m.qkv_width(), qw = m.q_width();
    const bool actor = mid == ACTOR;
    float* lm_master = actor ? m.lm_master : nullptr;
    mt.embed = make_pt(e, m.embed, V, D, true, d.tied ? lm_master : nullptr, st);
    if (!d.tied && actor) mt.lm_head = make_pt(e, m.lm_head, V, D, true, lm_master, st);
    else mt.lm_head = mt.embed;
    mt.final_norm = make_pt(e, m.final_norm, D, 1, false, nullptr, st);
    if (m.head) mt.head = make_pt(e, m.head, D, 1, false, nullptr, st);
    mt.layers.resize(d.n_layers);
    for (int l = 0; l < d.n_layers; ++l) {
        auto& L = m.layers[l];
        auto& T = mt.layers[l];
        T.wqkv = make_pt(e, L.wqkv, qkv, D, true, nullptr, st);
        T.bqkv = make_pt(e, L.bqkv, qkv, 1, false, nullptr, st);
        T.wo = make_pt(e, L.wo, D, qw, true, nullptr, st);
        T.wgu = make_pt(e, L.wgu, 2 * F, D, true, nullptr, st);
        T.wdown = make_pt(e, L.wdown, D, F, true, nullptr, st);
        T.ln1 = make_pt(e, L.ln1, D, 1, false, nullptr, st);
        T.ln2 = make_pt(e, L.ln2, D, 1, false, nullptr, st);
    }
    mt.ready = true;
}

// Y[M, N] (epilogue ep) = A[M, K] . B[N, K]^T, packed rows
void mm(Engine& e, cudaStream_t st, const void* A, int M, int K, const void* B, int N, EpiParams ep) {
    ep.update_gemm = 1;
    gemm_run(e, e.ws, st, A, M, K, K, B, N, K, ep);
}
// The same with operands read in place: K-major (kK, stored [M][K] / [N][K])
// or MN-major (kMN, stored [K][M] / [K][N]), leading dimension ld.
constexpr int kK = 0, kMN = 1;
void mmt(Engine& e, cudaStream_t st, const void* A, int a_mn, int lda, const void* B, int b_mn, int ldb, int M,
         int N, int K, EpiParams ep) {
    ep.pair_long_k = 1;  // long-K gradient GEMMs may take CTA-pair tiles
    ep.update_gemm = 1;
    gemm_run_t(e, e.ws, st, A, a_mn, lda, B, b_mn, ldb, M, N, K, ep);
}
EpiParams epi(int mode, void* y, int ldy, float scale = 1.f, const float* bias = nullptr) {
    EpiParams p{};
    p.mode = mode;
    p.y = y;
    p.ldy = ldy;
    p.scale = scale;
    p.bias = bias;
    return p;
}

// RMSNorm backward (dx += ..., bf16 copy into dxc when set) + gamma gradient
// (gout += column sums of dy * xh) in one pass, block partials in ts.colp.
template <class T>
void rms_bwd_into(TrainState& ts, const float* x, const float* g, const float* dy, int rows, int d, float* dx,
                  T* dxc, float* gout, cudaStream_t st) {
    if (rows <= 0) return;
    const int nblk = std::min(kColParts, std::max(1, rows / 16));  // 2 rows per warp at 32K rows
    const int per = cdiv(rows, nblk);
    const size_t smem = 8 * static_cast<size_t>(d) * 4;
    static bool attr = false;
    if (!attr) {
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(train::rms_bwd_cs<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024));
        attr = true;
    }
    train::rms_bwd_cs<T><<<nblk, 256, smem, st>>>(x, g, dy, rows, d, per, kEps, dx, dxc, ts.colp);
    train::colsum_final<<<cdiv(d, 32), 256, 0, st>>>(ts.colp, nblk, d, gout);
}

// y = x rounded to T and out += column sums of x, in one pass over x
template <class T>
void cvt_colsum_into(TrainState& ts, const float* x, int rows, int cols, T* y, float* out, cudaStream_t st) {
    if (rows <= 0) return;
    const int chunks = std::min(kColParts, std::max(1, rows / 64));
    const int per = cdiv(rows, chunks);
    train::cvt_colsum_part<T><<<dim3(cdiv(cols, 256), chunks), 256, 0, st>>>(x, rows, cols, per, y, ts.colp);
    train::colsum_final<<<cdiv(cols, 32), 256, 0, st>>>(ts.colp, chunks, cols, out);
}

void colsum_into(TrainState& ts, const float* x, int rows, int cols, float* out, cudaStream_t st) {
    if (rows <= 0) return;
    const int chunks = std::min(64, std::max(1, rows / 64));
    const int per = cdiv(rows, chunks);
    train::colsum_part<<<dim3(cdiv(cols, 256), chunks), 256, 0, st>>>(x, rows, cols, cols, per, ts.colp);
    train::colsum_final<<<cdiv(cols, 32), 256, 0, st>>>(ts.colp, chunks, cols, out);
}

template <class T>
void rmsnorm(Engine& e, float* x, const float* g, T* out, int rows, int D, cudaStream_t st,
             const float* head_w = nullptr, float* head_out = nullptr) {
    rmsnorm_rows<T><<<cdiv(rows, 4), 128, 0, st>>>(x, g, out, rows, D, kEps, head_w, head_out, nullptr, nullptr,
                                                   nullptr, 0, 0, -1, nullptr, 0, size_t(0));
}

template <class T>
void cvt_f32(const float* in, T* out, int64_t n, cudaStream_t st) {
    convert<float, T><<<cdiv(n, 256), 256, 0, st>>>(in, out, n);
}

template <class T, int HD>
void attn_launch(int which, const train::TBlk* blks, int nb, const T* qkv, int ld, int H, int KV, T* o, float* lse,
                 const T* dO, const float* dvec, float* dqkv, cudaStream_t st) {
    using A = train::AttnT<HD>;
    static bool attr = false;
    if (!attr) {
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(train::attn_train_fwd<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             A::SMEM_FWD));
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(train::attn_train_dq<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             A::SMEM_BWD));
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(train::attn_train_dkv<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             A::SMEM_BWD));
        attr = true;
    }
    if (which == 0)
        train::attn_train_fwd<T, HD><<<dim3(nb, H), 256, A::SMEM_FWD, st>>>(blks, qkv, ld, H, KV, o, lse);
    else if (which == 1)
        train::attn_train_dq<T, HD><<<dim3(nb, H), 256, A::SMEM_BWD, st>>>(blks, qkv, ld, H, KV, dO, lse, dvec, dqkv, ld);
    else
        train::attn_train_dkv<T, HD><<<dim3(nb, KV), 256, A::SMEM_BWD, st>>>(blks, qkv, ld, H, KV, dO, lse, dvec, dqkv, ld);
}
template <int HD>
void attn_mma_launch(int which, const train::TBlk* blks, int nb, const __nv_bfloat16* qkv, int ld, int H, int KV,
                     __nv_bfloat16* o, float* lse, const __nv_bfloat16* dO, const float* dvec, float* dqkv,
                     cudaStream_t st, float* part, int rows) {
    using M = train::MmaT<HD>;
    static bool attr = false;
    if (!attr) {
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(train::attn_fwd_mma<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             M::SMEM_FWD));
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(train::attn_dq_mma<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             M::SMEM_DQ));
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(train::attn_dkv_mma<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             M::SMEM_DKV));
        attr = true;
    }
    if (which == 0)
        train::attn_fwd_mma<HD><<<dim3(nb, H), 128, M::SMEM_FWD, st>>>(blks, qkv, ld, H, KV, o, lse);
    else if (which == 1)  // dq / dk come out with the RoPE transpose applied
        train::attn_dq_mma<HD><<<dim3(nb, H), 128, M::SMEM_DQ, st>>>(blks, qkv, ld, H, KV, dO, lse, dvec, dqkv, ld,
                                                                     kTheta);
    else {  // the G query heads of each KV head over G CTAs, then the ordered sum
        const int gs = part ? H / KV : 1;
        train::attn_dkv_mma<HD><<<dim3(nb, KV * gs), 128, M::SMEM_DKV, st>>>(blks, qkv, ld, H, KV, dO, lse, dvec, dqkv,
                                                                         ld, gs, part, rows, kTheta);
        if (gs > 1) {
            const int64_t n4 = static_cast<int64_t>(rows) * 2 * KV * HD / 4;
            train::dkv_combine<<<cdiv(n4, 256), 256, 0, st>>>(part, gs, rows, 2 * KV * HD, dqkv, ld, H * HD);
        }
    }
}

// tensor-core (mma.sync) attention for bf16 with head_dim 64 / 128 (64-row
// blocks), the SIMT kernels otherwise (fp32 engine, head_dim 32; 32-row blocks)
template <class T>
constexpr bool use_mma_attn(int hd) {
    return std::is_same_v<T, __nv_bfloat16> && (hd == 64 || hd == 128);
}

template <class T>
void attn(int hd, int which, const train::TBlk* blks, int nb, const T* qkv, int ld, int H, int KV, T* o, float* lse,
          const T* dO, const float* dvec, float* dqkv, cudaStream_t st, float* part = nullptr, int rows = 0) {
    if (nb <= 0) return;
    if constexpr (std::is_same_v<T, __nv_bfloat16>) {
        if (use_mma_attn<T>(hd) && std::getenv("OPPO_TRAIN_SIMT_ATTN") == nullptr) {
            if (hd == 64) attn_mma_launch<64>(which, blks, nb, qkv, ld, H, KV, o, lse, dO, dvec, dqkv, st, part, rows);
            else attn_mma_launch<128>(which, blks, nb, qkv, ld, H, KV, o, lse, dO, dvec, dqkv, st, part, rows);
            return;
        }
    }
    switch (hd) {
    case 32: attn_launch<T, 32>(which, blks, nb, qkv, ld, H, KV, o, lse, dO, dvec, dqkv, st); break;
    case 64: attn_launch<T, 64>(which, blks, nb, qkv, ld, H, KV, o, lse, dO, dvec, dqkv, st); break;
    default: attn_launch<T, 128>(which, blks, nb, qkv, ld, H, KV, o, lse, dO, dvec, dqkv, st); break;
    }
}

// Sizes the scratch for `rows` training rows of the largest trained model.
template <class T>
void ensure_scratch(Engine& e, TrainState& ts, int rows) {
    const int resp_rows = rows;  // a micro-batch never has more response rows than rows
    int L = 0, D = 0, qkv = 0, qw = 0, F = 0, H = 0, V = 0;
    for (int mid : {ACTOR, CRITIC}) {
        const Model& m = e.models[mid];
        L = std::max(L, m.dims.n_layers);
        D = std::max(D, m.dims.d_model);
        qkv = std::max(qkv, m.qkv_width());
        qw = std::max(qw, m.q_width());
        F = std::max(F, m.dims.d_ff);
        H = std::max(H, m.dims.n_heads);
        V = std::max(V, m.dims.vocab);
    }
    if (rows <= ts.rows_cap) return;
    ts.scr.release();
    for (auto* v : {&ts.x_in, &ts.x_mid, &ts.lse, &ts.rstd1, &ts.rstd2}) v->assign(L, nullptr);
    for (auto* v : {&ts.h1, &ts.h2, &ts.qkv, &ts.o, &ts.gu, &ts.ff}) v->assign(L, nullptr);
    const size_t R = rows, es = sizeof(T);
    for (int l = 0; l < L; ++l) {
        ts.x_in[l] = static_cast<float*>(ts.scr.take(R * D * 4));
        ts.x_mid[l] = static_cast<float*>(ts.scr.take(R * D * 4));
        ts.lse[l] = static_cast<float*>(ts.scr.take(R * H * 4));
        ts.rstd1[l] = static_cast<float*>(ts.scr.take(R * 4));
        ts.rstd2[l] = static_cast<float*>(ts.scr.take(R * 4));
        ts.h1[l] = ts.scr.take(R * D * es);
        ts.h2[l] = ts.scr.take(R * D * es);
        ts.qkv[l] = ts.scr.take(R * qkv * es);
        ts.o[l] = ts.scr.take(R * qw * es);
        ts.gu[l] = ts.scr.take(R * 2 * F * es);
        ts.ff[l] = ts.scr.take(R * F * es);
    }
    const size_t wide = std::max<size_t>({static_cast<size_t>(D), static_cast<size_t>(qkv), static_cast<size_t>(2 * F)});
    ts.x = static_cast<float*>(ts.scr.take(R * D * 4));
    ts.dx = static_cast<float*>(ts.scr.take(R * D * 4));
    ts.dh = static_cast<float*>(ts.scr.take(R * D * 4));
    ts.dqkv = static_cast<float*>(ts.scr.take(R * qkv * 4));
    size_t part_floats = 0;
    for (int mid : {ACTOR, CRITIC}) {
        const auto& md = e.models[mid].dims;
        part_floats = std::max(part_floats, static_cast<size_t>(md.n_heads / md.n_kv_heads) * R * 2 * md.n_kv_heads *
                                                md.head_dim);
    }
    ts.dkv_part = static_cast<float*>(ts.scr.take(part_floats * 4));
    ts.dvec = static_cast<float*>(ts.scr.take(R * H * 4));
    ts.gscr = static_cast<float*>(ts.scr.take(R * std::max(D, qkv) * 4));
    ts.colp = static_cast<float*>(ts.scr.take(kColParts * wide * 4));
    ts.head_out = static_cast<float*>(ts.scr.take(R * 4));
    ts.hf = ts.scr.take(R * D * es);
    ts.dgu = ts.scr.take(R * 2 * F * es);
    ts.dxc = ts.scr.take(R * D * es);
    ts.dO = ts.scr.take(R * qw * es);
    ts.dqkvc = ts.scr.take(R * qkv * es);
    ts.tok = static_cast<int32_t*>(ts.scr.take(R * 4));
    ts.pos = static_cast<int32_t*>(ts.scr.take(R * 4));
    ts.hf_resp = ts.scr.take(static_cast<size_t>(resp_rows) * D * es);
    ts.dhf_c = static_cast<float*>(ts.scr.take(static_cast<size_t>(resp_rows) * D * 4));
    ts.g_rows = std::min(resp_rows, 4096);
    ts.Gt = ts.scr.take(static_cast<size_t>(ts.g_rows) * V * es);
    ts.rows_cap = rows;
}

}  // namespace

// ----------------------------------------------------------------------
// One model's update over the batch (actor: clipped surrogate through the
// lm_head; critic: squared error of the value head).  Gradients accumulate
// into the tensors' fp32 grad buffers; the caller applies them.
template <class T>
void train_model(Engine& e, const TrainBatch& b, int mid, cudaStream_t st,
                 const std::function<void(int)>& layer_final = {}) {
    auto& ts = *static_cast<TrainState*>(e.train_state);
    Model& m = e.models[mid];
    ModelT& mt = ts.m[mid];
    const auto& d = m.dims;
    const int D = d.d_model, H = d.n_heads, KV = d.n_kv_heads, hd = d.head_dim, F = d.d_ff, V = d.vocab;
    const int qkvw = m.qkv_width(), qw = m.q_width(), Lyr = d.n_layers;
    const bool actor = mid == ACTOR;
    for (PT* p : mt.all()) OPPO_CUDA_CHECK(cudaMemsetAsync(p->grad, 0, p->n() * 4, st));
    // micro-batches of whole sequences
    const int n = static_cast<int>(b.slot.size());
    int s0 = 0;
    while (s0 < n) {
        int s1 = s0, rows = 0;
        while (s1 < n && (rows + b.P[s1] + b.L[s1] - 1 <= b.rows_max || s1 == s0)) {
            rows += b.P[s1] + b.L[s1] - 1;
            ++s1;
        }
        const int Tr = rows;
        const int r0 = b.off[s0], Nr = b.off[s1] - r0;  // response tokens of this micro-batch
        // metadata: sequences, attention blocks, response-row map
        std::vector<train::TSeq> seqs;
        std::vector<train::TBlk> blks;
        std::vector<int32_t> map;
        int row = 0;
        const int blk = (use_mma_attn<T>(hd) && std::getenv("OPPO_TRAIN_SIMT_ATTN") == nullptr) ? train::kMBlk
                                                                                              : train::kBlk;
        for (int i = s0; i < s1; ++i) {
            const int len = b.P[i] + b.L[i] - 1;
            seqs.push_back({b.slot[i], b.P[i], row, len});
            for (int q0 = 0; q0 < len; q0 += blk) blks.push_back({row, len, q0, 0});
            for (int j = 0; j < b.L[i]; ++j) map.push_back(row + b.P[i] - 1 + j);
            row += len;
        }
        std::vector<uint8_t> host;
        auto put = [&](const void* p, size_t bytes) {
            const size_t o = (host.size() + 255) & ~size_t(255);
            host.resize(o + bytes);
            std::memcpy(host.data() + o, p, bytes);
            return o;
        };
        const size_t o_seq = put(seqs.data(), seqs.size() * sizeof(train::TSeq));
        const size_t o_blk = put(blks.data(), blks.size() * sizeof(train::TBlk));
        const size_t o_map = put(map.data(), map.size() * 4);
        uint8_t* meta = static_cast<uint8_t*>(b.meta_dev);
        if (host.size() > b.meta_cap) internal_error("training metadata buffer too small");
        OPPO_CUDA_CHECK(cudaMemcpyAsync(meta, host.data(), host.size(), cudaMemcpyHostToDevice, st));
        const auto* d_seq = reinterpret_cast<const train::TSeq*>(meta + o_seq);
        const auto* d_blk = reinterpret_cast<const train::TBlk*>(meta + o_blk);
        const auto* d_map = reinterpret_cast<const int32_t*>(meta + o_map);
        const int nb = static_cast<int>(blks.size());
        train::train_rows<<<s1 - s0, 128, 0, st>>>(d_seq, e.d_prompt, e.Pmax, e.d_tok, e.tok_stride, ts.tok, ts.pos);
        // rows grouped by input token (CSR) for the deterministic embedding gradient
        std::vector<int32_t> toks(Tr);
        OPPO_CUDA_CHECK(cudaMemcpyAsync(toks.data(), ts.tok, Tr * 4, cudaMemcpyDeviceToHost, st));
        OPPO_CUDA_CHECK(cudaStreamSynchronize(st));  // also: `host` (pageable, local) has been read
        std::vector<int32_t> order(Tr);
        for (int r = 0; r < Tr; ++r) order[r] = r;
        std::stable_sort(order.begin(), order.end(), [&](int a, int c) { return toks[a] < toks[c]; });
        std::vector<int32_t> uniq, start;
        for (int k = 0; k < Tr; ++k)
            if (k == 0 || toks[order[k]] != toks[order[k - 1]]) {
                uniq.push_back(toks[order[k]]);
                start.push_back(k);
            }
        start.push_back(Tr);
        std::vector<uint8_t> host2;
        auto put2 = [&](const void* p, size_t bytes) {
            const size_t o = (host2.size() + 255) & ~size_t(255);
            host2.resize(o + bytes);
            std::memcpy(host2.data() + o, p, bytes);
            return o;
        };
        const size_t o_u = put2(uniq.data(), uniq.size() * 4), o_s = put2(start.data(), start.size() * 4),
                     o_r = put2(order.data(), order.size() * 4);
        const size_t base2 = (host.size() + 255) & ~size_t(255);
        if (base2 + host2.size() > b.meta_cap) internal_error("training metadata buffer too small");
        OPPO_CUDA_CHECK(cudaMemcpyAsync(meta + base2, host2.data(), host2.size(), cudaMemcpyHostToDevice, st));
        const auto* d_uniq = reinterpret_cast<const int32_t*>(meta + base2 + o_u);
        const auto* d_start = reinterpret_cast<const int32_t*>(meta + base2 + o_s);
        const auto* d_order = reinterpret_cast<const int32_t*>(meta + base2 + o_r);

        // ------------------------------------------------------- forward
        const bool rope_epi = std::is_same_v<T, __nv_bfloat16> && (hd == 64 || hd == 128) &&
                              std::getenv("OPPO_TRAIN_ROPE_KERNEL") == nullptr;
        float* x = ts.x;
        embed_rows<T><<<Tr, 128, 0, st>>>(static_cast<const T*>(m.embed), ts.tok, x, Tr, D);
        for (int l = 0; l < Lyr; ++l) {
            auto& Lw = m.layers[l];
            T* qkv = static_cast<T*>(ts.qkv[l]);
            T* o = static_cast<T*>(ts.o[l]);
            T* h1 = static_cast<T*>(ts.h1[l]);
            T* h2 = static_cast<T*>(ts.h2[l]);
            OPPO_CUDA_CHECK(cudaMemcpyAsync(ts.x_in[l], x, static_cast<size_t>(Tr) * D * 4, cudaMemcpyDeviceToDevice, st));
            train::rms_fwd_train<T><<<cdiv(Tr, 4), 128, 0, st>>>(x, Lw.ln1, Tr, D, kEps, h1, ts.rstd1[l]);
            if (rope_epi) {  // bias, bf16 round and RoPE of q, k in the projection's epilogue
                EpiParams er = epi(EPI_ROPE_APPEND, nullptr, qkvw, 1.f, Lw.bqkv);
                er.q_out = qkv;
                er.kv.head_dim = hd;
                er.kv.kv_heads = KV;
                er.n_heads = H;
                er.theta = kTheta;
                er.pos = ts.pos;
                mm(e, st, h1, Tr, D, Lw.wqkv, qkvw, er);
            } else {
                mm(e, st, h1, Tr, D, Lw.wqkv, qkvw, epi(EPI_STORE, qkv, qkvw, 1.f, Lw.bqkv));
                train::rope_rows<T><<<Tr, 128, 0, st>>>(qkv, qkvw, Tr, ts.pos, H + KV, hd, kTheta, 0);
            }
            attn<T>(hd, 0, d_blk, nb, qkv, qkvw, H, KV, o, ts.lse[l], nullptr, nullptr, nullptr, st);
            mm(e, st, o, Tr, qw, Lw.wo, D, epi(EPI_ADD_F32, x, D));
            OPPO_CUDA_CHECK(cudaMemcpyAsync(ts.x_mid[l], x, static_cast<size_t>(Tr) * D * 4, cudaMemcpyDeviceToDevice, st));
            train::rms_fwd_train<T><<<cdiv(Tr, 4), 128, 0, st>>>(x, Lw.ln2, Tr, D, kEps, h2, ts.rstd2[l]);
            EpiParams eg = epi(EPI_SWIGLU, ts.ff[l], F);  // SwiGLU product + saved (gate, up)
            eg.y2 = ts.gu[l];
            eg.ldy2 = 2 * F;
            mm(e, st, h2, Tr, D, Lw.wgu, 2 * F, eg);
            mm(e, st, ts.ff[l], Tr, F, Lw.wdown, D, epi(EPI_ADD_F32, x, D));
        }
        T* hf = static_cast<T*>(ts.hf);
        rmsnorm<T>(e, x, m.final_norm, hf, Tr, D, st, actor ? nullptr : m.head, ts.head_out);

        // ------------------------------------------------------- loss head
        float* d_hf = ts.dh;  // dObj / d(final normed hidden), fp32 [Tr, D]
        OPPO_CUDA_CHECK(cudaMemsetAsync(d_hf, 0, static_cast<size_t>(Tr) * D * 4, st));
        if (actor) {
            T* hr = static_cast<T*>(ts.hf_resp);
            train::gather_rows_t<T><<<Nr, 128, 0, st>>>(hf, d_map, Nr, D, hr);
            const int nt = gemm_logit_tiles(e.dtype, V);
            Work& w = e.ws;
            const int lrows = std::max(32, std::min(w.max_rows, static_cast<int>((static_cast<size_t>(64) << 20) / (nt * 16))));
            for (int c0 = 0; c0 < Nr; c0 += lrows) {  // current-policy log-probs of the sampled tokens
                const int cn = std::min(lrows, Nr - c0);
                EpiParams ep{};
                ep.mode = EPI_LOGITS;
                ep.partials = w.partials;
                ep.tgt_logit = w.tgt_logit;
                ep.targets = b.tok + r0 + c0;
                mm(e, st, hr + static_cast<size_t>(c0) * D, cn, D, m.lm_head, V, ep);
                logits_combine<<<cdiv(cn, 4), 128, 0, st>>>(w.partials, nt, V, cn, nullptr, w.tgt_logit, nullptr,
                                                            nullptr, nullptr, b.new_lp + r0 + c0, 0,
                                                            b.lse + r0 + c0, nullptr);
            }
            // K10 clipped objective + dObj/dlogp over this micro-batch's tokens
            const int cb = std::min(1024, std::max(1, cdiv(Nr, 256)));
            ppo_clip<float><<<cb, 256, 0, st>>>(Nr, b.new_lp + r0, b.old_lp + r0, b.adv + r0, b.clip_eps, b.stats,
                                                1e-8, b.dobj + r0, b.part, b.inv_n);
            sum_partials_acc<<<1, 32, 0, st>>>(b.part, cb, b.obj_acc);
            // dObj/dlogits = dobj * (onehot - softmax) in chunks: lm_head wgrad
            // and the hidden-state dgrad
            const PT& lm = mt.lm_head;
            for (int c0 = 0; c0 < Nr; c0 += ts.g_rows) {
                const int cn = std::min(ts.g_rows, Nr - c0);
                EpiParams ep{};  // G = dObj/dlogits [cn][V], row-major
                ep.mode = EPI_SOFTMAX_GRAD;
                ep.y2 = ts.Gt;
                ep.ldy2 = V;
                ep.lse = b.lse + r0 + c0;
                ep.coef = b.dobj + r0 + c0;
                ep.targets = b.tok + r0 + c0;
                const T* hc = hr + static_cast<size_t>(c0) * D;
                mm(e, st, hc, cn, D, m.lm_head, V, ep);
                // dW_lm += G^T H (both MN-major over the chunk's tokens); dH = G W_lm (W MN-major)
                mmt(e, st, ts.Gt, kMN, V, hc, kMN, D, V, D, cn, epi(EPI_ADD_F32, lm.grad, D));
                mmt(e, st, ts.Gt, kK, V, m.lm_head, kMN, D, cn, D, V, epi(EPI_STORE_F32, ts.dhf_c, D));
                train::scatter_rows_f<<<cn, 128, 0, st>>>(ts.dhf_c, d_map + c0, cn, D, d_hf);
            }
        } else {
            // K12 value regression toward the returns: (1/2N) sum (V - R)^2
            train::value_loss_grad<T><<<Nr, 128, 0, st>>>(ts.head_out, hf, d_map, Nr, D, b.ret + r0, m.head, b.inv_n,
                                                          d_hf, ts.gscr, b.sq + r0, b.v_new ? b.v_new + r0 : nullptr);
            colsum_into(ts, ts.gscr, Nr, D, mt.head.grad, st);
        }

        // ------------------------------------------------------- backward
        float* dx = ts.dx;
        T* dxc = static_cast<T*>(ts.dxc);  // dx rounded to T: the next GEMMs' operand
        OPPO_CUDA_CHECK(cudaMemsetAsync(dx, 0, static_cast<size_t>(Tr) * D * 4, st));
        rms_bwd_into<T>(ts, x, m.final_norm, d_hf, Tr, D, dx, dxc, mt.final_norm.grad, st);
        T* dgu = static_cast<T*>(ts.dgu);
        for (int l = Lyr - 1; l >= 0; --l) {
            auto& Lw = m.layers[l];
            auto& Lt = mt.layers[l];
            T* qkv = static_cast<T*>(ts.qkv[l]);
            // down projection (x += ff Wd^T, Wd [D][F]) and SwiGLU: the dgrad
            // GEMM's epilogue turns d ff into d(gate, up) from the saved pre-activations
            mmt(e, st, dxc, kMN, D, ts.ff[l], kMN, F, D, F, Tr, epi(EPI_ADD_F32, Lt.wdown.grad, F));
            EpiParams es = epi(EPI_SWIGLU_BWD, dgu, 2 * F);
            es.aux = ts.gu[l];
            mmt(e, st, dxc, kK, D, Lw.wdown, kMN, F, Tr, F, D, es);
            // gate|up projection (gu = h2 Wgu^T, Wgu [2F][D])
            mmt(e, st, dgu, kMN, 2 * F, ts.h2[l], kMN, D, 2 * F, D, Tr, epi(EPI_ADD_F32, Lt.wgu.grad, D));
            mmt(e, st, dgu, kK, 2 * F, Lw.wgu, kMN, D, Tr, D, 2 * F, epi(EPI_STORE_F32, ts.dh, D));
            rms_bwd_into<T>(ts, ts.x_mid[l], Lw.ln2, ts.dh, Tr, D, dx, dxc, Lt.ln2.grad, st);
            // O projection (x += o Wo^T, Wo [D][qw]) + attention
            mmt(e, st, dxc, kMN, D, ts.o[l], kMN, qw, D, qw, Tr, epi(EPI_ADD_F32, Lt.wo.grad, qw));
            T* dO = static_cast<T*>(ts.dO);
            mmt(e, st, dxc, kK, D, Lw.wo, kMN, qw, Tr, qw, D, epi(EPI_STORE, dO, qw));
            train::attn_dvec<T><<<cdiv(static_cast<int64_t>(Tr) * H * 32, 256), 256, 0, st>>>(
                dO, static_cast<const T*>(ts.o[l]), Tr, H, hd, ts.dvec);
            attn<T>(hd, 1, d_blk, nb, qkv, qkvw, H, KV, nullptr, ts.lse[l], dO, ts.dvec, ts.dqkv, st);
            attn<T>(hd, 2, d_blk, nb, qkv, qkvw, H, KV, nullptr, ts.lse[l], dO, ts.dvec, ts.dqkv, st,
                    std::getenv("OPPO_TRAIN_DKV_NOSPLIT") ? nullptr : ts.dkv_part, Tr);
            if (!use_mma_attn<T>(hd) || std::getenv("OPPO_TRAIN_SIMT_ATTN"))  // (the mma kernels rotate back)
                train::rope_rows<float><<<Tr, 128, 0, st>>>(ts.dqkv, qkvw, Tr, ts.pos, H + KV, hd, kTheta, 1);
            T* dqc = static_cast<T*>(ts.dqkvc);
            cvt_colsum_into<T>(ts, ts.dqkv, Tr, qkvw, dqc, Lt.bqkv.grad, st);  // bf16 operand + bias gradient
            // q|k|v projection (qkv = h1 Wqkv^T + b, Wqkv [qkv][D])
            mmt(e, st, dqc, kMN, qkvw, ts.h1[l], kMN, D, qkvw, D, Tr, epi(EPI_ADD_F32, Lt.wqkv.grad, D));
            mmt(e, st, dqc, kK, qkvw, Lw.wqkv, kMN, D, Tr, D, qkvw, epi(EPI_STORE_F32, ts.dh, D));
            rms_bwd_into<T>(ts, ts.x_in[l], Lw.ln1, ts.dh, Tr, D, dx, l > 0 ? dxc : static_cast<T*>(nullptr),
                            Lt.ln1.grad, st);
            if (layer_final && s1 == n) layer_final(l);  // layer l's gradients are final
        }
        train::embed_grad_csr<<<static_cast<int>(uniq.size()), 128, 0, st>>>(dx, d_uniq, d_start, d_order, D,
                                                                              mt.embed.grad);
        OPPO_CUDA_CHECK(cudaGetLastError());
        OPPO_CUDA_CHECK(cudaStreamSynchronize(st));  // host2 (pageable, local) has been read
        e.launches += 26 * Lyr + 20;
        s0 = s1;
    }
}

template <class T>
void sgd_into(PT* p, float scale, cudaStream_t st) {
    if (p->master)
            train::sgd_apply<T><<<cdiv(p->n(), 256), 256, 0, st>>>(p->master, p->grad, p->n(), scale, static_cast<T*>(p->w));
        else
            train::sgd_apply<T><<<cdiv(p->n(), 256), 256, 0, st>>>(static_cast<float*>(p->w), p->grad, p->n(), scale,
                                                                    static_cast<T*>(nullptr));
}

template <class T>
void train_apply(Engine& e, int mid, float scale, bool dp, cudaStream_t st) {
    auto& ts = *static_cast<TrainState*>(e.train_state);
    for (PT* p : ts.m[mid].all()) {
        if (dp) dp_allreduce_pub(e, p->grad, p->n(), false, st);
        sgd_into<T>(p, scale, st);
    }
    OPPO_CUDA_CHECK(cudaGetLastError());
}

// One bucket on the comm stream once the compute stream has produced it:
// grouped allreduce, then the SGD step of each tensor.
template <class T>
void bucket_apply(Engine& e, TrainState& ts, const std::vector<PT*>& ps, float scale, cudaStream_t st) {
    OPPO_CUDA_CHECK(cudaEventRecord(ts.ev_ready, st));
    OPPO_CUDA_CHECK(cudaStreamWaitEvent(ts.comm, ts.ev_ready, 0));
    std::vector<std::pair<float*, int64_t>> bufs;
    for (PT* p : ps) bufs.emplace_back(p->grad, p->n());
    dp_allreduce_bucket(e, bufs, ts.comm);
    for (PT* p : ps) sgd_into<T>(p, scale, ts.comm);
    OPPO_CUDA_CHECK(cudaGetLastError());
}

// train_model + train_apply with the data-parallel gradient buckets
// overlapped with the backward (NCCL communicator only).
template <class T>
void train_and_apply(Engine& e, TrainBatch& b, int mid, float scale, bool dp, cudaStream_t st) {
    auto& ts = *static_cast<TrainState*>(e.train_state);
    if (!dp || !e.nccl || std::getenv("OPPO_GRAD_BUCKETS_OFF")) {
        train_model<T>(e, b, mid, st);
        train_apply<T>(e, mid, scale, dp, st);
        return;
    }
    if (!ts.comm) {
        OPPO_CUDA_CHECK(cudaStreamCreateWithFlags(&ts.comm, cudaStreamNonBlocking));
        OPPO_CUDA_CHECK(cudaEventCreateWithFlags(&ts.ev_ready, cudaEventDisableTiming));
        OPPO_CUDA_CHECK(cudaEventCreateWithFlags(&ts.ev_comm, cudaEventDisableTiming));
    }
    ModelT& mt = ts.m[mid];
    train_model<T>(e, b, mid, st, [&](int l) {
        auto& L = mt.layers[l];
        bucket_apply<T>(e, ts, {&L.wqkv, &L.bqkv, &L.wo, &L.wgu, &L.wdown, &L.ln1, &L.ln2}, scale, st);
    });
    std::vector<PT*> rest{&mt.embed};
    if (mt.lm_head.w && mt.lm_head.w != mt.embed.w) rest.push_back(&mt.lm_head);
    rest.push_back(&mt.final_norm);
    if (mt.head.w) rest.push_back(&mt.head);
    bucket_apply<T>(e, ts, rest, scale, st);
    OPPO_CUDA_CHECK(cudaEventRecord(ts.ev_comm, ts.comm));
    OPPO_CUDA_CHECK(cudaStreamWaitEvent(st, ts.ev_comm, 0));  // updated weights before anything else
}

template <class T>
void train_full(Engine& e, TrainBatch& b, const oppo_ppo_hparams& hp, bool dp, cudaStream_t st) {
    if (!e.train_state) e.train_state = new TrainState();
    auto& ts = *static_cast<TrainState*>(e.train_state);
    setup_model(e, ts, ACTOR, st);
    setup_model(e, ts, CRITIC, st);
    int max_seq = 0;
    for (size_t i = 0; i < b.slot.size(); ++i) max_seq = std::max(max_seq, b.P[i] + b.L[i] - 1);
    b.rows_max = std::max(b.rows_max, max_seq);
    ensure_scratch<T>(e, ts, b.rows_max);
    if (hp.learning_rate != 0)  // ascent (ppo.cpp:288-290)
        train_and_apply<T>(e, b, ACTOR, static_cast<float>(hp.learning_rate), dp, st);
    if (hp.value_learning_rate != 0)  // descent on (V-R)^2/2
        train_and_apply<T>(e, b, CRITIC, -static_cast<float>(hp.value_learning_rate), dp, st);
}

// Every tensor the full update changes, for checkpoints: (device pointer,
// bytes) of the compute tensors and fp32 masters of the actor and critic.
std::vector<std::pair<void*, size_t>> train_tensors(Engine& e, cudaStream_t st) {
    if (!e.train_state) e.train_state = new TrainState();
    auto& ts = *static_cast<TrainState*>(e.train_state);
    std::vector<std::pair<void*, size_t>> out;
    for (int mid : {ACTOR, CRITIC}) {
        setup_model(e, ts, mid, st);
        for (PT* p : ts.m[mid].all()) {
            out.emplace_back(p->w, static_cast<size_t>(p->n()) * (p->matrix ? e.esz : 4));
            if (p->master) out.emplace_back(p->master, static_cast<size_t>(p->n()) * 4);
        }
    }
    OPPO_CUDA_CHECK(cudaStreamSynchronize(st));
    return out;
}

const float* train_master(Engine& e, int model, const std::string& name, int layer) {
    auto* ts = static_cast<TrainState*>(e.train_state);
    if (!ts || model < 0 || model >= N_MODELS || !ts->m[model].ready) return nullptr;
    ModelT& m = ts->m[model];
    PT* p = nullptr;
    if (name == "embed") p = &m.embed;
    else if (name == "lm_head") p = &m.lm_head;
    else if (layer >= 0 && layer < static_cast<int>(m.layers.size())) {
        auto& L = m.layers[layer];
        if (name == "wqkv") p = &L.wqkv;
        else if (name == "wo") p = &L.wo;
        else if (name == "wgu") p = &L.wgu;
        else if (name == "wdown") p = &L.wdown;
    }
    return p ? p->master : nullptr;
}

template void train_full<float>(Engine&, TrainBatch&, const oppo_ppo_hparams&, bool, cudaStream_t);
template void train_full<__nv_bfloat16>(Engine&, TrainBatch&, const oppo_ppo_hparams&, bool, cudaStream_t);

}  // namespace oppo
