// engine.cu — the GPU step executor behind oppo_run_step / oppo_ppo_update.
//
// One engine per GPU holds four Qwen2-style models (actor, reward, critic,
// reference), a paged KV cache per model sharing one page table, per-slot
// rollout buffers, and two streams:
//   sa (high priority): actor — prompt prefill at admission, then one lockstep
//       decode iteration per tick of the logical clock;
//   ss (low priority): scorers — chunk "waves" of reward / critic / reference
//       incremental prefill, each gated by an event recorded after the decode
//       iteration that completed the chunk (streamed mode), or one wave after
//       generation (sequential mode = overlap off).
// The cut (stop_after-th finisher), chunk boundaries and carried progress come
// from plan_step() (host), i.e. the reference's run_step under the lockstep
// latency model; the GPU realises exactly that work.
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <exception>
#include <functional>
#include <thread>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include <nccl.h>

#include "engine.cuh"
#include "host/driver.hpp"
#include "kernels/ppo.cuh"
#include "kernels/train.cuh"

namespace oppo {

namespace {

constexpr float kRmsEps = 1e-6f;
constexpr float kRopeTheta = 1e6f;

template <class T> constexpr int dtype_of();
template <> constexpr int dtype_of<float>() { return OPPO_DTYPE_F32; }
template <> constexpr int dtype_of<__nv_bfloat16>() { return OPPO_DTYPE_BF16; }

void* dalloc(size_t bytes) {
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    OPPO_CUDA_CHECK(cudaMalloc(&p, bytes));
    return p;
}

inline int cdiv(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// ------------------------------------------------------------ arena upload
struct Arena {  // one pinned host staging buffer -> one device buffer per step
    std::vector<uint8_t> host;
    void* dev = nullptr;
    size_t cap = 0;
    uint8_t* pinned = nullptr;
    size_t pinned_cap = 0;
    cudaEvent_t copied = nullptr;  // the last upload's H2D copy (pinned staging reuse)
    size_t push(const void* p, size_t bytes) {
        const size_t off = (host.size() + 255) & ~size_t(255);
        host.resize(off + bytes);
        if (bytes) std::memcpy(host.data() + off, p, bytes);
        return off;
    }
    template <class V> size_t push_vec(const std::vector<V>& v) {
        return push(v.data(), v.size() * sizeof(V));
    }
    template <class V> V* at(size_t off) { return reinterpret_cast<V*>(static_cast<uint8_t*>(dev) + off); }
    void upload(cudaStream_t st) {
        if (host.size() > cap) {
            if (dev) cudaFree(dev);
            cap = host.size() * 2;
            dev = dalloc(cap);
        }
        if (copied) OPPO_CUDA_CHECK(cudaEventSynchronize(copied));  // staging no longer read
        else OPPO_CUDA_CHECK(cudaEventCreateWithFlags(&copied, cudaEventDisableTiming));
        if (host.size() > pinned_cap) {
            if (pinned) cudaFreeHost(pinned);
            pinned_cap = host.size() * 2;
            OPPO_CUDA_CHECK(cudaMallocHost(&pinned, pinned_cap));
        }
        std::memcpy(pinned, host.data(), host.size());
        if (!host.empty())
            OPPO_CUDA_CHECK(cudaMemcpyAsync(dev, pinned, host.size(), cudaMemcpyHostToDevice, st));
        OPPO_CUDA_CHECK(cudaEventRecord(copied, st));
    }
    void release() {
        if (dev) cudaFree(dev);
        if (pinned) cudaFreeHost(pinned);
        if (copied) cudaEventDestroy(copied);
        copied = nullptr;
        dev = nullptr;
        pinned = nullptr;
        cap = pinned_cap = 0;
    }
};

// K13 flags.  wait_ready: the scorer wave's first kernel, one thread polling
// its flag (ld.acquire.gpu, cyclic >=; traps after 30 s instead of hanging);
// set_ready: a release store on the actor stream after the decode iteration
// that completed the wave's chunks.
__global__ void wait_ready(const uint32_t* __restrict__ flag, uint32_t want) {
    if (threadIdx.x != 0) return;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (static_cast<int32_t>(v - want) >= 0) break;
        __nanosleep(256);
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 30000000000ull) __trap();
    }
}
__global__ void set_ready(uint32_t* __restrict__ flag, uint32_t v) {
    if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}
bool eager_module_loading() {
    using Fn = CUresult (*)(CUmoduleLoadingMode*);
    static const bool eager = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuModuleGetLoadingMode", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return false;
        CUmoduleLoadingMode m;
        return reinterpret_cast<Fn>(p)(&m) == CUDA_SUCCESS && m == CU_MODULE_EAGER_LOADING;
    }();
    return eager;
}

// Host thread that enqueues the scorer waves on the scorer stream.  A wave is
// hundreds of launches; enqueued from the driver thread they can fill the
// launch queue and block it, starving the actor stream of its next decode
// graph.  With this thread the driver only records the wave's event on the
// actor stream and posts the wave here.  drain() ends every run_step, so the
// engine's API stays single-threaded.
struct ScorerWorker {
    std::thread th;
    std::mutex mu;
    std::condition_variable cv, cv_idle;
    std::deque<std::function<void()>> q;
    bool stop = false, busy = false, started = false;
    std::exception_ptr err;
    void start(int device) {
        if (started) return;
        started = true;
        th = std::thread([this, device] {
            cudaSetDevice(device);
            for (;;) {
                std::function<void()> job;
                {
                    std::unique_lock<std::mutex> lk(mu);
                    cv.wait(lk, [&] { return stop || !q.empty(); });
                    if (q.empty()) return;  // stop requested and nothing left
                    job = std::move(q.front());
                    q.pop_front();
                    busy = true;
                }
                try {
                    job();
                } catch (...) {
                    std::lock_guard<std::mutex> lk(mu);
                    if (!err) err = std::current_exception();
                }
                {
                    std::lock_guard<std::mutex> lk(mu);
                    busy = false;
                }
                cv_idle.notify_all();
            }
        });
    }
    void post(std::function<void()> f) {
        {
            std::lock_guard<std::mutex> lk(mu);
            q.push_back(std::move(f));
        }
        cv.notify_one();
    }
    void drain() {
        std::unique_lock<std::mutex> lk(mu);
        cv_idle.wait(lk, [&] { return q.empty() && !busy; });
        if (err) {
            std::exception_ptr x = err;
            err = nullptr;
            std::rethrow_exception(x);
        }
    }
    void shutdown() {
        {
            std::lock_guard<std::mutex> lk(mu);
            stop = true;
        }
        cv.notify_all();
        if (th.joinable()) th.join();
    }
};

struct EngineExtra {
    Arena step_arena, admit_arena, upd_arena;
    ScorerWorker scorer;
};
std::unordered_map<const Engine*, EngineExtra> g_extra;

int env_int(const char* k, int dflt) {
    const char* v = std::getenv(k);
    return v ? std::atoi(v) : dflt;
}

template <class F>
F driver_fn(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
        throw Error(OPPO_ERR_CUDA, std::string(name) + " unavailable");
    return reinterpret_cast<F>(p);
}

#define OPPO_CU_CHECK(x)                                                                    \
    do {                                                                                    \
        const CUresult r_ = (x);                                                            \
        if (r_ != CUDA_SUCCESS)                                                             \
            throw Error(OPPO_ERR_CUDA, std::string(#x) + " failed (" + std::to_string(r_) + ")"); \
    } while (0)

// Fixed SM partition (north_star: "concurrent streams with a fixed SM
// partition"): two green contexts on the device, `scorer_sms` SMs (rounded up
// to the architecture's granularity of 8) for the reward/critic/reference
// prefill and the rest for the actor's decode.  Each stream is created inside
// its green context, so kernels launched on it only run on its SMs; memory is
// shared with the primary context.
void make_sm_partition(Engine& e, int scorer_sms, int prio_hi, int prio_lo) {
    using GetDev = CUresult (*)(CUdevice*, int);
    using GetRes = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
    using Split = CUresult (*)(CUdevResource*, unsigned int*, const CUdevResource*, CUdevResource*,
                               unsigned int, unsigned int);
    using GenDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned int);
    using GCreate = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned int);
    using GStream = CUresult (*)(CUstream*, CUgreenCtx, unsigned int, int);
    CUdevice dev;
    OPPO_CU_CHECK(driver_fn<GetDev>("cuDeviceGet")(&dev, e.cfg.device));
    CUdevResource all{}, grp{}, rest{};
    OPPO_CU_CHECK(driver_fn<GetRes>("cuDeviceGetDevResource")(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    unsigned int n = 1;
    // OPPO_SPLIT_FLAGS: CUdevSmResourceSplit_flags (cluster-friendly layout was
    // tried for CTA-pair GEMMs inside the scorer partition; they hang there)
    const unsigned flags = static_cast<unsigned>(env_int("OPPO_SPLIT_FLAGS", 0));
    OPPO_CU_CHECK(driver_fn<Split>("cuDevSmResourceSplitByCount")(&grp, &n, &all, &rest, flags,
                                                                  static_cast<unsigned>(scorer_sms)));
    if (n != 1 || rest.sm.smCount == 0) config_error("SM partition: scorer_sms leaves no actor SMs");
    CUdevResourceDesc ds, da;
    OPPO_CU_CHECK(driver_fn<GenDesc>("cuDevResourceGenerateDesc")(&ds, &grp, 1));
    OPPO_CU_CHECK(driver_fn<GenDesc>("cuDevResourceGenerateDesc")(&da, &rest, 1));
    OPPO_CU_CHECK(driver_fn<GCreate>("cuGreenCtxCreate")(&e.gctx_scorer, ds, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    OPPO_CU_CHECK(driver_fn<GCreate>("cuGreenCtxCreate")(&e.gctx_actor, da, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream a, a2, s, s1, s2;
    OPPO_CU_CHECK(driver_fn<GStream>("cuGreenCtxStreamCreate")(&s1, e.gctx_scorer, CU_STREAM_NON_BLOCKING, prio_lo));
    OPPO_CU_CHECK(driver_fn<GStream>("cuGreenCtxStreamCreate")(&s2, e.gctx_scorer, CU_STREAM_NON_BLOCKING, prio_lo));
    e.ss_m[0] = reinterpret_cast<cudaStream_t>(s1);
    e.ss_m[1] = reinterpret_cast<cudaStream_t>(s2);
    OPPO_CU_CHECK(driver_fn<GStream>("cuGreenCtxStreamCreate")(&a, e.gctx_actor, CU_STREAM_NON_BLOCKING, prio_hi));
    OPPO_CU_CHECK(driver_fn<GStream>("cuGreenCtxStreamCreate")(&a2, e.gctx_actor, CU_STREAM_NON_BLOCKING, prio_hi));
    OPPO_CU_CHECK(driver_fn<GStream>("cuGreenCtxStreamCreate")(&s, e.gctx_scorer, CU_STREAM_NON_BLOCKING, prio_lo));
    e.sa = reinterpret_cast<cudaStream_t>(a);
    e.sa2 = reinterpret_cast<cudaStream_t>(a2);
    e.ss = reinterpret_cast<cudaStream_t>(s);
    e.sms_actor = static_cast<int>(rest.sm.smCount);
    e.sms_scorer = static_cast<int>(grp.sm.smCount);
}

// --------------------------------------------------------------- weights
template <class T>
void init_tensor(T* p, int64_t n, uint64_t seed, uint64_t id, float std_, cudaStream_t st) {
    if (n <= 0) return;
    init_normal<T><<<cdiv(n, 256), 256, 0, st>>>(p, n, seed, id, std_);
}
template <class T>
void fill_tensor(T* p, int64_t n, float v, cudaStream_t st) {
    if (n <= 0) return;
    fill_value<T><<<cdiv(n, 256), 256, 0, st>>>(p, n, v);
}

template <class T>
void build_model(Engine& e, Model& m, int id, cudaStream_t st) {
    const auto& d = m.dims;
    const uint64_t seed = e.cfg.weight_seed;
    auto tid = [&](int layer, int t) {
        return (static_cast<uint64_t>(id) << 40) | (static_cast<uint64_t>(layer + 1) << 8) | t;
    };
    const int64_t V = d.vocab, D = d.d_model;
    m.embed = dalloc(V * D * sizeof(T));
    init_tensor(static_cast<T*>(m.embed), V * D, seed, tid(-1, 0), 0.02f, st);
    if (d.tied) {
        m.lm_head = m.embed;
    } else {
        m.lm_head = dalloc(V * D * sizeof(T));
        init_tensor(static_cast<T*>(m.lm_head), V * D, seed, tid(-1, 1), 0.02f, st);
    }
    const int64_t qkv = m.qkv_width(), qw = m.q_width(), F = d.d_ff;
    m.layers.resize(d.n_layers);
    for (int l = 0; l < d.n_layers; ++l) {
        auto& L = m.layers[l];
        L.wqkv = dalloc(qkv * D * sizeof(T));
        L.bqkv = static_cast<float*>(dalloc(qkv * sizeof(float)));
        L.wo = dalloc(D * qw * sizeof(T));
        L.wgu = dalloc(2 * F * D * sizeof(T));
        L.wdown = dalloc(D * F * sizeof(T));
        L.ln1 = static_cast<float*>(dalloc(D * sizeof(float)));
        L.ln2 = static_cast<float*>(dalloc(D * sizeof(float)));
        init_tensor(static_cast<T*>(L.wqkv), qkv * D, seed, tid(l, 1), 0.02f, st);
        init_tensor(L.bqkv, qkv, seed, tid(l, 2), 0.02f, st);
        init_tensor(static_cast<T*>(L.wo), D * qw, seed, tid(l, 3), 0.02f, st);
        init_tensor(static_cast<T*>(L.wgu), 2 * F * D, seed, tid(l, 4), 0.02f, st);
        init_tensor(static_cast<T*>(L.wdown), D * F, seed, tid(l, 5), 0.02f, st);
        fill_tensor(L.ln1, D, 1.0f, st);
        fill_tensor(L.ln2, D, 1.0f, st);
    }
    m.final_norm = static_cast<float*>(dalloc(D * sizeof(float)));
    fill_tensor(m.final_norm, D, 1.0f, st);
    if (id == REWARD || id == CRITIC) {
        m.head = static_cast<float*>(dalloc(D * sizeof(float)));
        init_tensor(m.head, D, seed, tid(-1, 7), id == REWARD ? 0.5f : 0.02f, st);
    }
    // KV pools
    m.layer_stride = static_cast<int64_t>(e.n_pages + 1) * d.n_kv_heads * e.page_size * d.head_dim;
    const size_t kvb = static_cast<size_t>(m.layer_stride) * d.n_layers * sizeof(T);
    m.k_pool = dalloc(kvb);
    m.v_pool = dalloc(kvb);
    OPPO_CUDA_CHECK(cudaMemsetAsync(m.k_pool, 0, kvb, st));
    OPPO_CUDA_CHECK(cudaMemsetAsync(m.v_pool, 0, kvb, st));
    m.used = true;
}

void check_dims(const oppo_model_dims& d, const char* who) {
    auto bad = [&](const std::string& m) { config_error(std::string(who) + ": " + m); };
    if (d.d_model > 32 * 4 * 28) bad("d_model above 3584 is not supported by rmsnorm_rows");
    if (d.n_layers < 1 || d.d_model < 64 || d.d_model % 64) bad("d_model must be a multiple of 64");
    if (d.n_heads < 1 || d.n_kv_heads < 1 || d.n_heads % d.n_kv_heads)
        bad("n_heads must be a multiple of n_kv_heads");
    if (d.head_dim != 32 && d.head_dim != 64 && d.head_dim != 128) bad("head_dim must be 32/64/128");
    if (d.d_ff < 64 || d.d_ff % 64) bad("d_ff must be a multiple of 64");
    if (d.vocab < 2) bad("vocab must be >= 2");
    if ((d.n_heads * d.head_dim) % 64) bad("n_heads*head_dim must be a multiple of 64");
}

template <class T>
void alloc_work(Engine& e, Work& w, int rows, bool lm_rows) {
    int dmax = 0, qkvmax = 0, qmax = 0, fmax_ = 0, vmax = 0, hmax = 0, hdmax = 0;
    for (auto& m : e.models) {
        if (!m.used) continue;
        dmax = std::max(dmax, m.dims.d_model);
        qkvmax = std::max(qkvmax, m.qkv_width());
        qmax = std::max(qmax, m.q_width());
        fmax_ = std::max(fmax_, m.dims.d_ff);
        vmax = std::max(vmax, m.dims.vocab);
        hmax = std::max(hmax, m.dims.n_heads);
        hdmax = std::max(hdmax, m.dims.head_dim);
    }
    w.max_rows = rows;
    const size_t R = rows;
    w.meta.slot = static_cast<int32_t*>(dalloc(R * 4));
    w.meta.pos = static_cast<int32_t*>(dalloc(R * 4));
    w.meta.tok = static_cast<int32_t*>(dalloc(R * 4));
    w.meta.t = static_cast<int32_t*>(dalloc(R * 4));
    w.meta.key = static_cast<uint64_t*>(dalloc(R * 8));
    w.x = static_cast<float*>(dalloc(R * dmax * 4));
    w.h = dalloc(R * dmax * sizeof(T));
    w.qkv = dalloc(R * qkvmax * sizeof(T));
    w.q = dalloc(R * qmax * sizeof(T));
    w.attn = dalloc(R * qmax * sizeof(T));
    w.ff = dalloc(R * fmax_ * sizeof(T));
    w.head_out = static_cast<float*>(dalloc(R * 4));
    const int lm_R = lm_rows ? rows : rows;
    w.partials = static_cast<float4*>(dalloc(static_cast<size_t>(lm_R) * gemm_logit_tiles(dtype_of<T>(), vmax) * 16));
    w.tgt_logit = static_cast<float*>(dalloc(R * 4));
    w.lse = static_cast<float*>(dalloc(R * 4));
    w.lm_in = dalloc(R * dmax * sizeof(T));
    w.lm_tgt = static_cast<int32_t*>(dalloc(R * 4));
    w.lm_slot = static_cast<int32_t*>(dalloc(R * 4));
    w.lm_t = static_cast<int32_t*>(dalloc(R * 4));
    w.gemm_ws_floats = static_cast<size_t>(16) << 20;  // 64 MB
    w.gemm_ws = static_cast<float*>(dalloc(w.gemm_ws_floats * 4));
    w.gemm_cnt_n = 1 << 16;
    w.gemm_cnt = static_cast<int*>(dalloc(w.gemm_cnt_n * 4));
    OPPO_CUDA_CHECK(cudaMemset(w.gemm_cnt, 0, w.gemm_cnt_n * 4));
    w.attn_ws_rows = std::max<size_t>(R * hmax * 8, static_cast<size_t>(e.num_sms) * 64);
    w.attn_ws_o = static_cast<float*>(dalloc(w.attn_ws_rows * hdmax * 4));
    w.attn_ws_ml = static_cast<float*>(dalloc(w.attn_ws_rows * 2 * 4));
}

void free_work(Work& w) {
    for (void* p : {static_cast<void*>(w.meta.slot), static_cast<void*>(w.meta.pos), static_cast<void*>(w.meta.tok),
                    static_cast<void*>(w.meta.t), static_cast<void*>(w.meta.key), static_cast<void*>(w.x), w.h,
                    w.qkv, w.q, w.attn, w.ff, static_cast<void*>(w.head_out), static_cast<void*>(w.partials),
                    static_cast<void*>(w.tgt_logit), static_cast<void*>(w.lse), w.lm_in,
                    static_cast<void*>(w.lm_tgt), static_cast<void*>(w.lm_slot), static_cast<void*>(w.lm_t),
                    static_cast<void*>(w.gemm_ws), static_cast<void*>(w.gemm_cnt), static_cast<void*>(w.attn_ws_o),
                    static_cast<void*>(w.attn_ws_ml)})
        if (p) cudaFree(p);
    w = Work{};
}

// --------------------------------------------------------------- forward
template <class T>
void launch_attn_decode(bool pdl, int hd, int G, dim3 grid, cudaStream_t st, const T* q, T* out,
                        const KvView& kv, int layer, const int32_t* slot, const int32_t* pos,
                        int rows, int split_len, float* wo, float* wml) {
#define OPPO_ATTN(HD_, G_)                                                                   \
    if (hd == HD_ && G == G_) {                                                              \
        launch(pdl, attn_decode<T, HD_, G_>, grid, dim3(128), 0, st, q, out, kv, layer, slot,   \
               pos, rows, split_len, wo, wml);                                               \
        return;                                                                              \
    }
    OPPO_ATTN(32, 1)
    OPPO_ATTN(32, 2)
    OPPO_ATTN(64, 1)
    OPPO_ATTN(64, 2)
    OPPO_ATTN(64, 7)
    OPPO_ATTN(128, 1)
    OPPO_ATTN(128, 6)
    OPPO_ATTN(128, 7)
#undef OPPO_ATTN
    config_error("unsupported (head_dim, q heads per kv head) = (" + std::to_string(hd) + ", " +
                 std::to_string(G) + ")");
}

template <class T>
void launch_attn_prefill(bool pdl, int hd, dim3 grid, cudaStream_t st, const T* q, T* out,
                         const KvView& kv, int layer, const QBlock* blocks, int n_heads) {
    if (hd == 32) launch(pdl, attn_prefill<T, 32>, grid, dim3(128), 0, st, q, out, kv, layer, blocks, n_heads);
    else if (hd == 64) launch(pdl, attn_prefill<T, 64>, grid, dim3(128), 0, st, q, out, kv, layer, blocks, n_heads);
    else launch(pdl, attn_prefill<T, 128>, grid, dim3(128), 0, st, q, out, kv, layer, blocks, n_heads);
}

void attn_mma_launch(Engine& e, const Model& m, Work& w, cudaStream_t st, int layer, int R,
                     bool decode, int splits, const QBlock* qblocks, int n_qblocks) {
    const auto& d = m.dims;
    const KvView kv = m.kv(e.d_page_table, e.max_pages, e.page_size);
    const auto* q = static_cast<const __nv_bfloat16*>(w.q);
    auto* o = static_cast<__nv_bfloat16*>(w.attn);
    // decode split-KV: the splits of one row form a cluster and merge in DSMEM
    const bool cluster = decode && splits > 1 && e.attn_cluster;
    auto go = [&](auto kernel, dim3 grid, int threads) {
        if (cluster)
            launch_cluster_z(e.pdl, splits, kernel, grid, dim3(threads), 0, st, q, o, kv, layer, d.n_heads,
                             w.meta.slot, w.meta.pos, R, static_cast<float*>(nullptr),
                             static_cast<float*>(nullptr), static_cast<const QBlock*>(nullptr));
        else
            launch(e.pdl, kernel, grid, dim3(threads), 0, st, q, o, kv, layer, d.n_heads, w.meta.slot,
                   w.meta.pos, R, w.attn_ws_o, w.attn_ws_ml, decode ? nullptr : qblocks);
    };
    const dim3 grid = decode ? dim3(R, d.n_kv_heads, splits) : dim3(n_qblocks, d.n_kv_heads);
    switch (d.head_dim) {
    case 32: decode ? go(attn_mma<32, 1>, grid, 32) : go(attn_mma<32, 4>, grid, 128); break;
    case 64: decode ? go(attn_mma<64, 1>, grid, 32) : go(attn_mma<64, 4>, grid, 128); break;
    default: decode ? go(attn_mma<128, 1>, grid, 32) : go(attn_mma<128, 4>, grid, 128); break;
    }
    if (decode && splits > 1 && !cluster) {
        launch(e.pdl, attn_split_combine<__nv_bfloat16>, dim3(R, d.n_heads), dim3(64), 0, st,
               w.attn_ws_o, w.attn_ws_ml, o, R, d.n_heads, d.head_dim, splits);
        e.launches += 1;
    }
}

// Decode attention with RoPE + KV append fused (attn_dec.cuh), bf16.  The
// qkv row comes from the decode GEMM's partials (n_part > 0) or a bf16 row.
template <int HD, int NW, int TPO = 0>
void attn_dec_launch_hd(Engine& e, const Model& m, Work& w, cudaStream_t st, int layer, int R,
                        const float* part, int n_part, const float* bias) {
    using Cf = AttnDecCfg<HD, NW, TPO>;
    static std::once_flag attr;
    std::call_once(attr, [] {
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(attn_dec<HD, NW, TPO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Cf::SMEM));
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(attn_dec<HD, NW, TPO>,
                                             cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    });
    const auto& d = m.dims;
    const KvView kv = m.kv(e.d_page_table, e.max_pages, e.page_size);
    const int base = R * d.n_kv_heads;
    // split-KV clusters for long-context iterations; each row uses only as
    // many of the cluster's CTAs as give it >= attn_split_minpos positions.
    // Measured (profiles/r02_attn_split.txt): 7B actor at ctx 2K, 16 rows,
    // iteration 7.15 -> 5.86 ms; 0.5B at ctx 768, 32-64 rows, -4..-5.5%; a
    // cluster launch at short contexts costs +5-16% (hence the host's
    // per-iteration choice between the two graph variants)
    // (only in long-context iterations, e.attn_long, and while the clustered
    // grid stays within 2 CTAs per SM: larger clustered grids measured slower)
    const int resident = std::max(1, std::min(2, (227 * 1024) / Cf::SMEM));  // CTAs per SM (shared memory)
    int nsp = std::max(1, std::min((resident * w.sms) / base, Cf::MAX_SPLIT));
    nsp = std::min(nsp, e.attn_max_split > 0 ? e.attn_max_split : 8);
    if (!e.attn_long) nsp = 1;
    const dim3 grid(R, d.n_kv_heads, nsp);
    auto* out = static_cast<__nv_bfloat16*>(w.attn);
    const auto* qkv = static_cast<const __nv_bfloat16*>(w.qkv);
    const size_t pstride = static_cast<size_t>(R) * m.qkv_width();
    // early K/V tile loads help while the grid is under one wave (latency);
    // with several waves they only add memory traffic to the critical fold
    const int early = base * nsp <= 2 * w.sms ? 1 : 0;
    const int smem = early ? Cf::SMEM : Cf::SMEM_ALIAS;
    if (nsp > 1)
        launch_cluster_z(e.pdl, nsp, attn_dec<HD, NW, TPO>, grid, dim3(Cf::THREADS), smem, st, part, n_part, pstride, bias,
                         qkv, out, kv, layer, d.n_heads, w.meta.slot, w.meta.pos, R, kRopeTheta, early,
                         e.attn_split_minpos);
    else
        launch(e.pdl, attn_dec<HD, NW, TPO>, grid, dim3(Cf::THREADS), smem, st, part, n_part, pstride, bias, qkv, out, kv,
               layer, d.n_heads, w.meta.slot, w.meta.pos, R, kRopeTheta, early, e.attn_split_minpos);
    e.launches += 1;
}

bool attn_dec_supported(const oppo_model_dims& d) {
    const int G = d.n_heads / d.n_kv_heads;
    return G <= 16 && (d.head_dim == 32 || d.head_dim == 64 || d.head_dim == 128);
}

void attn_dec_launch(Engine& e, const Model& m, Work& w, cudaStream_t st, int layer, int R,
                     const float* part, int n_part, const float* bias) {
    // 8 warps x 16-position tiles (head_dim <= 64) while the grid is within one
    // wave (measured -90 us per iteration at 16-128 rows), 4 warps x 32 above
    const bool w8 = e.attn_warps == 8 ||
                    (e.attn_warps == 0 && 10 * R * m.dims.n_kv_heads <= e.attn_w8_tenths * w.sms);
    switch (m.dims.head_dim) {
    case 32:
        if (w8) attn_dec_launch_hd<32, 8>(e, m, w, st, layer, R, part, n_part, bias);
        else attn_dec_launch_hd<32, 4>(e, m, w, st, layer, R, part, n_part, bias);
        break;
    case 64:
        if (w8) attn_dec_launch_hd<64, 8>(e, m, w, st, layer, R, part, n_part, bias);
        else if (e.attn_tp16 > 0 || (e.attn_tp16 < 0 && R * m.dims.n_kv_heads >= 5 * w.sms))
            attn_dec_launch_hd<64, 4, 16>(e, m, w, st, layer, R, part, n_part, bias);
        else attn_dec_launch_hd<64, 4>(e, m, w, st, layer, R, part, n_part, bias);
        break;
    default:
        // head_dim 128 (the 7B actor): 8 warps (149 KB, one CTA per SM) while
        // the unsplit grid fits one wave: twice the K/V tiles in flight per row
        if (e.attn_warps == 8 || (e.attn_warps == 0 && R * m.dims.n_kv_heads <= w.sms))
            attn_dec_launch_hd<128, 8>(e, m, w, st, layer, R, part, n_part, bias);
        else
            attn_dec_launch_hd<128, 4>(e, m, w, st, layer, R, part, n_part, bias);
        break;
    }
}

template <class T>
struct Final {
    bool write_h = true;
    const float* head = nullptr;
    T* cache = nullptr;  // per-slot hidden cache [S, tok_stride, d]
    int t_lo = 1, t_hi = 0;
};

template <class T>
void forward(Engine& e, Model& m, Work& w, cudaStream_t st, int R, bool decode, int max_ctx,
             const QBlock* qblocks, int n_qblocks, const Final<T>& fin) {
    const auto& d = m.dims;
    const int D = d.d_model, H = d.n_heads, KV = d.n_kv_heads, hd = d.head_dim;
    const KvView kv = m.kv(e.d_page_table, e.max_pages, e.page_size);
    launch(e.pdl, embed_rows<T>, dim3(R), dim3(128), 0, st, static_cast<const T*>(m.embed), w.meta.tok, w.x, R, D);
    const int nrm_blocks = cdiv(R, 4);
    int splits = 1, split_len = 0;  // 0: each row splits its own context (graph-stable)
    if (decode) {
        const int base = R * KV;
        // bf16: 1-warp CTAs, split into clusters of <= 8 (DSMEM merge) until
        // ~4 CTAs per SM; fp32 (parity path): workspace + combine kernel
        const int per_sm = e.attn_per_sm;
        const int max_split = e.attn_max_split > 0 ? e.attn_max_split
                              : (!std::is_same_v<T, __nv_bfloat16> || !e.attn_cluster) ? 16
                              : hd == 32 ? attn_merge_splits<32>()
                              : hd == 64 ? attn_merge_splits<64>() : attn_merge_splits<128>();
        splits = std::max(1, std::min(cdiv(per_sm * w.sms, base), max_split));
        while (splits > 1 && static_cast<size_t>(R) * H * splits > w.attn_ws_rows) --splits;
    }
    (void)max_ctx;
    // decode (bf16, <= 512 rows): swap-AB gemm_dec with split-K partials folded
    // by the consumer kernels (RoPE/KV append, RMSNorm residual add)
    const bool dec_gemm = std::is_same_v<T, __nv_bfloat16> && decode && R <= 512 && D <= 4096 &&
                          D % 64 == 0 && m.q_width() % 64 == 0 && d.d_ff % 64 == 0;
    if (dec_gemm) {
        const size_t rope_smem = static_cast<size_t>(m.qkv_width()) * sizeof(T);
        const float* part = w.gemm_ws;
        int np = 0;  // partial splits pending for the next RMSNorm (0: none)
        // Per-GEMM choice between the swap-AB decode GEMM (weight-streaming:
        // wins while the token count is small or K is long) and the
        // token-tiled GEMM (wins once ~128+ tokens re-read the weights);
        // crossovers measured on B200 (tools/gemm_bench.py, profiles/).
        auto residual = [&](const void* xin, int K, const void* wt) -> int {
            if (K >= 2048 || R <= e.dec_res_max)
                return gemm_dec_run(e, w, st, xin, R, K, K, wt, D, K, DEC_PARTIAL, nullptr, 0, nullptr);
            EpiParams ep{};
            ep.mode = EPI_ADD_F32;
            ep.y = w.x;
            ep.ldy = D;
            ep.scale = 1.f;
            gemm_run(e, w, st, xin, R, K, K, wt, D, K, ep);
            return 0;
        };
        // OPPO_DEBUG_SKIP (perf diagnosis only; results are garbage): bit 1
        // attention, 2 RoPE/KV append, 4 norms, 8 projection GEMMs
        const int skip = e.debug_skip;
        const bool fused_attn = e.attn_fused && attn_dec_supported(d);
        for (int l = 0; l < d.n_layers; ++l) {
            const auto& L = m.layers[l];
            if (!(skip & 4)) launch(e.pdl, residual_rmsnorm<T>, dim3(R), dim3(256), 0, st, w.x, L.ln1,
                   static_cast<T*>(w.h), R, D, kRmsEps, part, np, static_cast<size_t>(R) * D, nullptr,
                   nullptr, nullptr, nullptr, nullptr, 0, 0, -1);
            int sq = 0;
            if (skip & 8) {
            } else if (R <= e.dec_qkv_max) {
                sq = gemm_dec_run(e, w, st, w.h, R, D, D, L.wqkv, m.qkv_width(), D, DEC_PARTIAL, nullptr,
                                  0, nullptr);
            } else {
                EpiParams ep{};
                ep.mode = EPI_STORE;
                ep.y = w.qkv;
                ep.ldy = m.qkv_width();
                ep.bias = L.bqkv;
                ep.scale = 1.f;
                gemm_run(e, w, st, w.h, R, D, D, L.wqkv, m.qkv_width(), D, ep);
            }
            if (fused_attn) {  // RoPE + KV append + attention in one launch
                if (!(skip & 1)) attn_dec_launch(e, m, w, st, l, R, sq ? part : nullptr, sq, L.bqkv);
            } else {
                if (!(skip & 2)) launch(e.pdl, rope_append<T>, dim3(R), dim3(128), sq ? rope_smem : 0, st,
                       static_cast<const T*>(w.qkv), static_cast<T*>(w.q), kv, l, w.meta.slot, w.meta.pos, R,
                       H, kRopeTheta, sq ? part : nullptr, sq, static_cast<size_t>(R) * m.qkv_width(), L.bqkv);
                if (!(skip & 1)) attn_mma_launch(e, m, w, st, l, R, decode, splits, qblocks, n_qblocks);
                e.launches += 2;  // rope + attention
            }
            np = (skip & 8) ? 0 : residual(w.attn, m.q_width(), L.wo);
            if (!(skip & 4)) launch(e.pdl, residual_rmsnorm<T>, dim3(R), dim3(256), 0, st, w.x, L.ln2,
                   static_cast<T*>(w.h), R, D, kRmsEps, part, np, static_cast<size_t>(R) * D, nullptr,
                   nullptr, nullptr, nullptr, nullptr, 0, 0, -1);
            if (skip & 8) {
            } else if (R <= e.dec_gu_max) {
                gemm_dec_run(e, w, st, w.h, R, D, D, L.wgu, 2 * d.d_ff, D, DEC_SWIGLU, w.ff, d.d_ff, nullptr);
            } else {
                EpiParams ep{};
                ep.mode = EPI_SWIGLU;
                ep.y = w.ff;
                ep.ldy = d.d_ff;
                ep.scale = 1.f;
                gemm_run(e, w, st, w.h, R, D, D, L.wgu, 2 * d.d_ff, D, ep);
            }
            np = (skip & 8) ? 0 : residual(w.ff, d.d_ff, L.wdown);
            e.launches += 2;  // the two norms (GEMMs / attention count themselves)
        }
        launch(e.pdl, residual_rmsnorm<T>, dim3(R), dim3(256), 0, st, w.x, m.final_norm,
               fin.write_h ? static_cast<T*>(w.h) : nullptr, R, D, kRmsEps, part, np,
               static_cast<size_t>(R) * D, fin.head, w.head_out, fin.cache, w.meta.slot, w.meta.t,
               e.tok_stride, fin.t_lo, fin.t_hi);
        e.launches += 2;
        OPPO_CUDA_CHECK(cudaGetLastError());
        return;
    }
    const bool rope_epi = std::is_same_v<T, __nv_bfloat16> && e.rope_epi && (hd == 64 || hd == 128);
    for (int l = 0; l < d.n_layers; ++l) {
        const auto& L = m.layers[l];
        launch(e.pdl, rmsnorm_rows<T>, dim3(nrm_blocks), dim3(128), 0, st, w.x, L.ln1, static_cast<T*>(w.h), R, D, kRmsEps,
                                                    nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0, -1,
                                                    nullptr, 0, size_t(0));
        EpiParams ep{};
        ep.bias = L.bqkv;
        ep.scale = 1.f;
        if (rope_epi) {  // RoPE + KV append in the projection's epilogue
            ep.mode = EPI_ROPE_APPEND;
            ep.q_out = w.q;
            ep.kv = kv;
            ep.layer = l;
            ep.n_heads = H;
            ep.theta = kRopeTheta;
            ep.slot = w.meta.slot;
            ep.pos = w.meta.pos;
            gemm_run(e, w, st, w.h, R, D, D, L.wqkv, m.qkv_width(), D, ep);
            e.launches -= 1;  // counted below with the rope launch it replaces
        } else {
            ep.mode = EPI_STORE;
            ep.y = w.qkv;
            ep.ldy = m.qkv_width();
            gemm_run(e, w, st, w.h, R, D, D, L.wqkv, m.qkv_width(), D, ep);
            launch(e.pdl, rope_append<T>, dim3(R), dim3(128), 0, st, static_cast<const T*>(w.qkv),
                   static_cast<T*>(w.q), kv, l, w.meta.slot, w.meta.pos, R, H, kRopeTheta, nullptr, 0,
                   size_t(0), nullptr);
        }
        if constexpr (std::is_same_v<T, __nv_bfloat16>) {
            attn_mma_launch(e, m, w, st, l, R, decode, splits, qblocks, n_qblocks);
        } else if (decode) {
            launch_attn_decode<T>(e.pdl, hd, H / KV, dim3(R, KV, splits), st, static_cast<const T*>(w.q),
                                  static_cast<T*>(w.attn), kv, l, w.meta.slot, w.meta.pos, R,
                                  split_len, w.attn_ws_o, w.attn_ws_ml);
            if (splits > 1 && !std::is_same_v<T, __nv_bfloat16>)
                launch(e.pdl, attn_split_combine<T>, dim3(dim3(R, H)), dim3(64), 0, st, w.attn_ws_o, w.attn_ws_ml,
                                                                static_cast<T*>(w.attn), R, H, hd,
                                                                splits);
        } else {
            launch_attn_prefill<T>(e.pdl, hd, dim3(n_qblocks, H), st, static_cast<const T*>(w.q),
                                   static_cast<T*>(w.attn), kv, l, qblocks, H);
        }
        ep = EpiParams{};
        ep.mode = EPI_ADD_F32;
        ep.y = w.x;
        ep.ldy = D;
        ep.scale = 1.f;
        gemm_run(e, w, st, w.attn, R, m.q_width(), m.q_width(), L.wo, D, m.q_width(), ep);
        launch(e.pdl, rmsnorm_rows<T>, dim3(nrm_blocks), dim3(128), 0, st, w.x, L.ln2, static_cast<T*>(w.h), R, D, kRmsEps,
                                                    nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0, -1,
                                                    nullptr, 0, size_t(0));
        ep = EpiParams{};
        ep.mode = EPI_SWIGLU;
        ep.y = w.ff;
        ep.ldy = d.d_ff;
        ep.scale = 1.f;
        gemm_run(e, w, st, w.h, R, D, D, L.wgu, 2 * d.d_ff, D, ep);
        ep = EpiParams{};
        ep.mode = EPI_ADD_F32;
        ep.y = w.x;
        ep.ldy = D;
        ep.scale = 1.f;
        gemm_run(e, w, st, w.ff, R, d.d_ff, d.d_ff, L.wdown, D, d.d_ff, ep);
        e.launches += 6 + (splits > 1 && !std::is_same_v<T, __nv_bfloat16>);
    }
    launch(e.pdl, rmsnorm_rows<T>, dim3(nrm_blocks), dim3(128), 0, st, 
        w.x, m.final_norm, fin.write_h ? static_cast<T*>(w.h) : nullptr, R, D, kRmsEps, fin.head,
        w.head_out, fin.cache, w.meta.slot, w.meta.t, e.tok_stride, fin.t_lo, fin.t_hi,
        nullptr, 0, size_t(0));
    e.launches += 2;
    OPPO_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

// =================================================================== create
Engine* engine_new(const oppo_engine_cfg& cfg) {
    auto* e = new Engine();
    e->cfg = cfg;
    try {
        e->dtype = cfg.dtype;
        if (cfg.dtype != OPPO_DTYPE_F32 && cfg.dtype != OPPO_DTYPE_BF16)
            config_error("dtype must be f32 or bf16");
        e->esz = cfg.dtype == OPPO_DTYPE_F32 ? 4 : 2;
        const oppo_model_dims* dims[N_MODELS] = {&cfg.actor, &cfg.reward, &cfg.critic, &cfg.ref};
        const char* names[N_MODELS] = {"actor", "reward", "critic", "ref"};
        for (int i = 0; i < N_MODELS; ++i) {
            check_dims(*dims[i], names[i]);
            e->models[i].dims = *dims[i];
        }
        const int V = cfg.actor.vocab;
        if (cfg.ref.vocab != V) config_error("actor and ref must share one vocabulary");
        if (cfg.reward.vocab != V || cfg.critic.vocab != V)
            config_error("all models must share one vocabulary (SURVEY 2.4)");
        if (cfg.max_slots < 1) config_error("max_slots must be >= 1");
        if (cfg.max_prompt_len < 1 || cfg.max_response_len < 1)
            config_error("max prompt/response lengths must be >= 1");
        OPPO_CUDA_CHECK(cudaSetDevice(cfg.device));
        OPPO_CUDA_CHECK(cudaDeviceGetAttribute(&e->num_sms, cudaDevAttrMultiProcessorCount, cfg.device));
        int lo = 0, hi = 0;
        OPPO_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        OPPO_CUDA_CHECK(cudaFree(nullptr));  // make the primary context current
        e->sms_actor = e->sms_scorer = e->num_sms;
        const int split = cfg.scorer_sms > 0 ? cfg.scorer_sms : env_int("OPPO_SCORER_SMS", 0);
        if (split > 0) {
            make_sm_partition(*e, split, hi, lo);  // fixed SM split: scorers | actor
            OPPO_CUDA_CHECK(cudaStreamCreateWithPriority(&e->su, cudaStreamNonBlocking, hi));
        } else {
            OPPO_CUDA_CHECK(cudaStreamCreateWithPriority(&e->sa, cudaStreamNonBlocking, hi));
            OPPO_CUDA_CHECK(cudaStreamCreateWithPriority(&e->sa2, cudaStreamNonBlocking, hi));
            OPPO_CUDA_CHECK(cudaStreamCreateWithPriority(&e->ss, cudaStreamNonBlocking, lo));
            for (auto& sm : e->ss_m) OPPO_CUDA_CHECK(cudaStreamCreateWithPriority(&sm, cudaStreamNonBlocking, lo));
            e->su = e->sa;
        }
        for (cudaEvent_t* ev : {&e->ev_begin, &e->ev_dec_end, &e->ev_sc_end, &e->ev_done, &e->ev_loop0})
            OPPO_CUDA_CHECK(cudaEventCreate(ev));
        for (cudaEvent_t* ev : {&e->ev_fork, &e->ev_join, &e->ev_pre, &e->ev_seg, &e->ev_m[0], &e->ev_m[1],
                                 &e->ev_admit})
            OPPO_CUDA_CHECK(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));

        e->S = cfg.max_slots;
        e->Pmax = cfg.max_prompt_len;
        e->Lmax = cfg.max_response_len;
        e->page_size = cfg.page_size > 0 ? cfg.page_size : 64;
        e->max_pages = cdiv(e->Pmax + e->Lmax + 1, e->page_size);
        e->n_pages = cfg.kv_pages > 0 ? cfg.kv_pages : e->S * e->max_pages;
        // one scratch slot (index S) and page (index n_pages) absorb padded /
        // finished rows of bucketed decode graphs
        e->tok_stride = e->Lmax + 2;
        for (int s = e->S - 1; s >= 0; --s) e->free_slots.push_back(s);
        for (int p = e->n_pages - 1; p >= 0; --p) e->free_pages.push_back(p);
        e->slots.resize(e->S);

        const size_t S = e->S + 1, TS = e->tok_stride;
        e->d_page_table = static_cast<int32_t*>(dalloc(S * e->max_pages * 4));
        OPPO_CUDA_CHECK(cudaMemset(e->d_page_table, 0, S * e->max_pages * 4));
        e->d_prompt = static_cast<int32_t*>(dalloc(S * e->Pmax * 4));
        OPPO_CUDA_CHECK(cudaMemset(e->d_prompt, 0, S * e->Pmax * 4));  // incl. the scratch slot
        e->d_tok = static_cast<int32_t*>(dalloc(S * TS * 4));
        OPPO_CUDA_CHECK(cudaMemset(e->d_tok, 0, S * TS * 4));
        e->d_old_lp = static_cast<float*>(dalloc(S * TS * 4));
        e->d_ref_lp = static_cast<float*>(dalloc(S * TS * 4));
        e->d_values = static_cast<float*>(dalloc(S * TS * 4));
        OPPO_CUDA_CHECK(cudaMemset(e->d_values, 0, S * TS * 4));
        OPPO_CUDA_CHECK(cudaMemset(e->d_ref_lp, 0, S * TS * 4));
        e->d_reward = static_cast<float*>(dalloc(S * 4));
        e->d_dseq = static_cast<DecodeSeq*>(dalloc((S + 16) * sizeof(DecodeSeq)));
        {
            std::vector<int32_t> dummy_row(e->max_pages, e->n_pages);
            OPPO_CUDA_CHECK(cudaMemcpy(e->d_page_table + static_cast<size_t>(e->S) * e->max_pages,
                                       dummy_row.data(), e->max_pages * 4, cudaMemcpyHostToDevice));
        }
        e->d_iter = static_cast<int32_t*>(dalloc(64));
        e->d_target_len = static_cast<int32_t*>(dalloc(S * 4));
        e->d_hf_actor = dalloc(S * TS * cfg.actor.d_model * e->esz);
        e->d_hf_critic = dalloc(S * TS * cfg.critic.d_model * e->esz);
        e->d_ref_pending = dalloc(S * cfg.ref.d_model * e->esz);

        cudaStream_t st = e->sa;
        for (int i = 0; i < N_MODELS; ++i) {
            if (e->dtype == OPPO_DTYPE_F32) build_model<float>(*e, e->models[i], i, st);
            else build_model<__nv_bfloat16>(*e, e->models[i], i, st);
        }
        if (cfg.train_heads) {
            auto& a = e->models[ACTOR];
            const size_t n = static_cast<size_t>(a.dims.vocab) * a.dims.d_model;
            a.lm_master = static_cast<float*>(dalloc(n * 4));
            if (e->dtype == OPPO_DTYPE_F32)
                convert<float, float><<<cdiv(n, 256), 256, 0, st>>>(static_cast<float*>(a.lm_head), a.lm_master, n);
            else
                convert<__nv_bfloat16, float><<<cdiv(n, 256), 256, 0, st>>>(
                    static_cast<__nv_bfloat16*>(a.lm_head), a.lm_master, n);
        }
        e->prefill_rows = std::max(1024, std::min(8192, e->S * (e->Pmax + 64)));
        if (e->dtype == OPPO_DTYPE_BF16)
            for (const auto& m : e->models)
                e->qblock = std::min(e->qblock, 64 / (m.dims.n_heads / m.dims.n_kv_heads));
        if (e->dtype == OPPO_DTYPE_F32) {
            alloc_work<float>(*e, e->wa, std::max(e->S + 16, 32), false);
            alloc_work<float>(*e, e->ws, e->prefill_rows, true);
        } else {
            alloc_work<__nv_bfloat16>(*e, e->wa, std::max(e->S + 16, 32), false);
            alloc_work<__nv_bfloat16>(*e, e->ws, e->prefill_rows, true);
        }
        e->wa.sms = e->sms_actor;
        e->ws.sms = e->sms_scorer;
        // reward | critic | reference passes concurrently on three scorer streams:
        // score end 1145 -> 1119 ms per cfg2 step (profiles/r01_experiments.txt)
        e->scorer_streams = env_int("OPPO_SCORER_STREAMS", 3) >= 3 ? 3 : 1;
        for (int k = 0; k < 2 && e->scorer_streams == 3; ++k) {
            if (e->dtype == OPPO_DTYPE_F32) alloc_work<float>(*e, e->ws_m[k], e->prefill_rows, true);
            else alloc_work<__nv_bfloat16>(*e, e->ws_m[k], e->prefill_rows, true);
            e->ws_m[k].sms = e->sms_scorer;
        }
        // two-branch decode iterations (bf16): the rows split in halves that run
        // concurrently on sa / sa2, each half's launch latencies hidden behind
        // the other's kernels (the weights are streamed twice)
        e->dec_split_min = env_int("OPPO_DEC_SPLIT_MIN", 144);  // bench sweep 96/128/144/176/208: 144 best
        if (e->dec_split_min > 0 && e->dtype == OPPO_DTYPE_BF16) {
            alloc_work<__nv_bfloat16>(*e, e->wa2, std::max(e->S + 16, 32), false);
            e->wa2.sms = e->sms_actor;
        } else {
            e->dec_split_min = 0;
        }
        // OPPO_NUMERICS_SMS pins every SM-count-dependent kernel choice that
        // changes the arithmetic (split-K factors, attention tile shapes, grid
        // shares of the two decode branches) to one SM count, so engines with
        // and without the SM partition compute bit-identical results (test
        // knob; by default each stream plans for the SMs it runs on)
        if (const int ns = env_int("OPPO_NUMERICS_SMS", 0); ns > 0)
            for (Work* w : {&e->wa, &e->wa2, &e->ws, &e->ws_m[0], &e->ws_m[1]}) w->sms = ns;
        // persistent decode kernel: experimental, off by default (measured slower
        // than the PDL-chained kernels: 2 us per grid barrier x 168, profiles/)
        e->attn_cluster = env_int("OPPO_ATTN_CLUSTER", 1) != 0;
        e->attn_per_sm = std::max(1, env_int("OPPO_ATTN_PER_SM", 4));
        e->attn_max_split = env_int("OPPO_ATTN_MAX_SPLIT", 0);
        e->attn_split_minpos = std::max(1, env_int("OPPO_ATTN_SPLIT_MINPOS", 512));
        e->attn_long_ctx = std::max(1, env_int("OPPO_ATTN_LONG_CTX", 768));
        e->debug_skip = env_int("OPPO_DEBUG_SKIP", 0);
        e->attn_fused = env_int("OPPO_ATTN_FUSED", 1) != 0;
        e->lmhead_dec_max = env_int("OPPO_LMHEAD_DEC_MAX", 32);  // measured crossover ~40 rows
        e->attn_warps = env_int("OPPO_ATTN_WARPS", 0);  // 0 auto, 4 or 8 forced
        e->attn_w8_tenths = env_int("OPPO_ATTN_W8_TENTHS", 20);  // auto: 8 warps up to 2.0 CTAs/SM
        e->dec_qkv_max = env_int("OPPO_DEC_QKV_MAX", 96);
        e->rope_epi = env_int("OPPO_ROPE_EPI", 1) != 0;
        // off: with concurrent scorer passes the scorers finish within ~8 ms of
        // decode, shorter than the precompute on the actor SMs (215.4 vs 213.6)
        e->pre_lp = env_int("OPPO_PRE_LP", 0) != 0;
        e->prompt_t0 = env_int("OPPO_PROMPT_T0", 1) != 0;
        e->chunk_flags = env_int("OPPO_CHUNK_FLAGS", 1) != 0 && eager_module_loading();
        e->d_ready = static_cast<uint32_t*>(dalloc(Engine::kReadyRing * sizeof(uint32_t)));
        OPPO_CUDA_CHECK(cudaMemsetAsync(e->d_ready, 0, Engine::kReadyRing * sizeof(uint32_t), st));
        e->g_chunk = std::max(64, env_int("OPPO_G_CHUNK", e->g_chunk)) / 8 * 8;  // update token chunk
        // 16-position tiles (5 CTAs/SM instead of 3) once the 32-position grid
        // needs 2+ waves: measured -190 us per iteration at 256 rows on 84 SMs
        e->attn_tp16 = env_int("OPPO_ATTN_TP16", -1);
        e->dec_gu_max = env_int("OPPO_DEC_GU_MAX", 64);
        e->dec_res_max = env_int("OPPO_DEC_RES_MAX", 192);
        e->nccl = cfg.nccl_comm;
        e->pdl = cfg.use_graphs != 0 && env_int("OPPO_PDL", 1) != 0;
        OPPO_CUDA_CHECK(cudaStreamSynchronize(st));
        g_extra[e];
    } catch (...) {
        engine_free(e);
        throw;
    }
    return e;
}

void engine_free(Engine* e) {
    if (!e) return;
    cudaDeviceSynchronize();
    train_free(*e);
    auto it = g_extra.find(e);
    if (it != g_extra.end()) {
        it->second.scorer.shutdown();
        it->second.step_arena.release();
        it->second.admit_arena.release();
        it->second.upd_arena.release();
        g_extra.erase(it);
    }
    // device memory is reclaimed with the process/context; free the big pools explicitly
    for (auto& m : e->models) {
        if (!m.used) continue;
        cudaFree(m.k_pool);
        cudaFree(m.v_pool);
        for (auto& L : m.layers) {
            cudaFree(L.wqkv);
            cudaFree(L.bqkv);
            cudaFree(L.wo);
            cudaFree(L.wgu);
            cudaFree(L.wdown);
            cudaFree(L.ln1);
            cudaFree(L.ln2);
        }
        if (m.lm_head != m.embed) cudaFree(m.lm_head);
        cudaFree(m.embed);
        cudaFree(m.final_norm);
        if (m.head) cudaFree(m.head);
        if (m.lm_master) cudaFree(m.lm_master);
    }
    for (void* p : {static_cast<void*>(e->d_hf_actor), static_cast<void*>(e->d_hf_critic),
                    static_cast<void*>(e->d_ref_pending), e->g_buf, e->ht_buf, e->ppo_buf,
                    static_cast<void*>(e->g_lm), e->pre_hf, static_cast<void*>(e->pre_tok),
                    static_cast<void*>(e->pre_new), static_cast<void*>(e->pre_lse), static_cast<void*>(e->pre_meta),
                    static_cast<void*>(e->pre_partials), static_cast<void*>(e->pre_tgt),
                    static_cast<void*>(e->d_ready)})
        if (p) cudaFree(p);
    for (auto& kv : e->decode_graphs) cudaGraphExecDestroy(kv.second);
    for (Work* w : {&e->wa, &e->wa2, &e->ws, &e->ws_m[0], &e->ws_m[1]}) free_work(*w);
    for (cudaEvent_t ev : {e->ev_seg, e->ev_m[0], e->ev_m[1], e->ev_admit})
        if (ev) cudaEventDestroy(ev);
    for (cudaStream_t sm : e->ss_m)
        if (sm) cudaStreamDestroy(sm);
    for (cudaEvent_t ev : e->ev_wave) cudaEventDestroy(ev);
    for (cudaEvent_t ev : {e->ev_begin, e->ev_dec_end, e->ev_sc_end, e->ev_done, e->ev_loop0, e->ev_fork, e->ev_join,
                           e->ev_pre})
        if (ev) cudaEventDestroy(ev);
    if (e->su && e->su != e->sa) cudaStreamDestroy(e->su);
    if (e->sa2) cudaStreamDestroy(e->sa2);
    if (e->sa) cudaStreamDestroy(e->sa);
    if (e->ss) cudaStreamDestroy(e->ss);
    try {
        using GDestroy = CUresult (*)(CUgreenCtx);
        if (e->gctx_actor) driver_fn<GDestroy>("cuGreenCtxDestroy")(e->gctx_actor);
        if (e->gctx_scorer) driver_fn<GDestroy>("cuGreenCtxDestroy")(e->gctx_scorer);
    } catch (...) {
    }
    delete e;
    cudaGetLastError();  // teardown is best effort: leave no error for the caller's next CUDA call
}

// =================================================================== admit
namespace {

void open_step(Engine& e) {
    if (e.step_open) return;
    OPPO_CUDA_CHECK(cudaEventRecord(e.ev_begin, e.sa));
    e.step_open = true;
    e.launches = 0;
}

// The admission prefill and the PPO update run between decode loops on the
// whole-GPU stream su with the (prefill-sized) scorer workspace: size their
// grids for all SMs.
struct ActorSms {
    Work& w;
    int saved;
    explicit ActorSms(Engine& e) : w(e.ws), saved(e.ws.sms) { w.sms = e.num_sms; }
    ~ActorSms() { w.sms = saved; }
};

template <class T>
void admit_impl(Engine& e, const oppo_seq_state* seqs, int n, const int32_t* prompts) {
    open_step(e);
    ActorSms actor_sms(e);
    std::vector<int32_t> slots, lens;
    std::vector<int64_t> ids;
    std::vector<int32_t> pt_rows;  // page-table rows, S x max_pages layout subset
    std::vector<int32_t> tlen;
    // Validate the whole batch before touching any host state, so a rejected
    // admission leaves the engine exactly as it was (no half-registered
    // sequences pointing at stale device rows).
    {
        std::unordered_map<int64_t, int> seen;
        size_t pages_needed = 0, tot = 0;
        for (int i = 0; i < n; ++i) {
            const auto& s = seqs[i];
            if (e.slot_of.count(s.id) || seen.count(s.id))
                input_error("sequence " + std::to_string(s.id) + " already admitted");
            seen[s.id] = i;
            if (s.prompt_len < 1 || s.prompt_len > e.Pmax) input_error("prompt_len outside [1, max_prompt_len]");
            if (s.target_len < 1 || s.target_len > e.Lmax)
                input_error("target_len outside [1, max_response_len]");
            pages_needed += cdiv(s.prompt_len + s.target_len + 1, e.page_size);
            tot += s.prompt_len;
        }
        if (static_cast<size_t>(n) > e.free_slots.size()) input_error("no free slot (raise max_slots)");
        if (pages_needed > e.free_pages.size()) input_error("KV page pool exhausted");
        if (prompts) {
            const int V = e.models[ACTOR].dims.vocab;
            for (size_t i = 0; i < tot; ++i)
                if (prompts[i] < 0 || prompts[i] >= V) input_error("prompt token outside the vocabulary");
        }
    }
    for (int i = 0; i < n; ++i) {
        const auto& s = seqs[i];
        const int need = cdiv(s.prompt_len + s.target_len + 1, e.page_size);
        const int slot = e.free_slots.back();
        e.free_slots.pop_back();
        auto& info = e.slots[slot];
        info = SlotInfo{};
        info.id = s.id;
        info.prompt_len = s.prompt_len;
        info.target_len = s.target_len;
        for (int p = 0; p < need; ++p) {
            info.pages.push_back(e.free_pages.back());
            e.free_pages.pop_back();
        }
        e.slot_of[s.id] = slot;
        slots.push_back(slot);
        lens.push_back(s.prompt_len);
        ids.push_back(s.id);
        tlen.push_back(s.target_len);
    }
    if (n == 0) return;
    auto& A = g_extra[&e].admit_arena;
    A.host.clear();
    // page table rows
    std::vector<int32_t> rows(static_cast<size_t>(n) * e.max_pages, 0);
    for (int i = 0; i < n; ++i) {
        const auto& pg = e.slots[slots[i]].pages;
        std::copy(pg.begin(), pg.end(), rows.begin() + static_cast<size_t>(i) * e.max_pages);
    }
    const size_t o_rows = A.push_vec(rows), o_slots = A.push_vec(slots), o_lens = A.push_vec(lens),
                 o_ids = A.push_vec(ids), o_tlen = A.push_vec(tlen);
    size_t o_prompts = 0;
    if (prompts) {
        size_t tot = 0;
        for (int i = 0; i < n; ++i) tot += lens[i];
        o_prompts = A.push(prompts, tot * 4);
    }
    // actor prompt prefill: positions 0..P-2 (the last prompt token feeds decode step 1)
    std::vector<Segment> segs;
    std::vector<QBlock> qbs;
    int rows_total = 0;
    for (int i = 0; i < n; ++i) {
        const int np = lens[i] - 1;
        if (np <= 0) continue;
        segs.push_back({slots[i], 0, np, rows_total, lens[i], 0});
        for (int b = 0; b < np; b += e.qblock)
            qbs.push_back({rows_total + b, std::min(e.qblock, np - b), slots[i], b});
        rows_total += np;
    }
    // prefill in passes of <= ws.max_rows rows (segments are whole prompts);
    // every pass's metadata rides the one admission upload, so the passes run
    // back to back on su without host round trips
    Work& w = e.ws;  // the scorer workspace has prefill-sized buffers; the scorer stream is idle
    struct AdmitPass { size_t o_seg, o_qb; int n_seg, n_qb, rows; };
    std::vector<AdmitPass> passes;
    for (size_t si = 0; si < segs.size();) {
        size_t sj = si;
        int rows_pass = 0;
        while (sj < segs.size() && (rows_pass + segs[sj].n <= w.max_rows || sj == si)) {
            rows_pass += segs[sj].n;
            ++sj;
        }
        if (rows_pass > w.max_rows) input_error("prompt longer than the prefill workspace");
        std::vector<Segment> ps(segs.begin() + si, segs.begin() + sj);
        std::vector<QBlock> pq;
        const int base = segs[si].row0;
        for (auto& sg : ps) sg.row0 -= base;
        for (const auto& q : qbs)
            if (q.row0 >= base && q.row0 < base + rows_pass) {
                QBlock bq = q;
                bq.row0 -= base;
                pq.push_back(bq);
            }
        passes.push_back({A.push_vec(ps), A.push_vec(pq), static_cast<int>(ps.size()),
                          static_cast<int>(pq.size()), rows_pass});
        si = sj;
    }
    A.upload(e.su);
    cudaStream_t st = e.su;  // admission prefill: whole GPU
    for (int i = 0; i < n; ++i)
        OPPO_CUDA_CHECK(cudaMemcpyAsync(e.d_page_table + static_cast<size_t>(slots[i]) * e.max_pages,
                                        A.at<int32_t>(o_rows) + static_cast<size_t>(i) * e.max_pages,
                                        e.max_pages * 4, cudaMemcpyDeviceToDevice, st));
    for (int i = 0; i < n; ++i)  // target lengths, scattered by slot
        OPPO_CUDA_CHECK(cudaMemcpyAsync(e.d_target_len + slots[i], A.at<int32_t>(o_tlen) + i, 4,
                                        cudaMemcpyDeviceToDevice, st));
    if (prompts) {
        size_t off = 0;
        for (int i = 0; i < n; ++i) {
            OPPO_CUDA_CHECK(cudaMemcpyAsync(e.d_prompt + static_cast<size_t>(slots[i]) * e.Pmax,
                                            A.at<int32_t>(o_prompts) + off, lens[i] * 4,
                                            cudaMemcpyDeviceToDevice, st));
            off += lens[i];
        }
    } else {
        prompt_tokens<<<n, 128, 0, st>>>(e.d_prompt, e.Pmax, A.at<int32_t>(o_slots),
                                         A.at<int64_t>(o_ids), A.at<int32_t>(o_lens), n,
                                         e.cfg.sample_seed, e.models[ACTOR].dims.vocab);
    }
    for (const auto& ap : passes) {
        segment_rows<<<ap.n_seg, 128, 0, st>>>(A.at<Segment>(ap.o_seg), e.d_prompt, e.Pmax, e.d_tok,
                                               e.tok_stride, w.meta);
        Final<T> fin;
        fin.write_h = false;
        forward<T>(e, e.models[ACTOR], w, st, ap.rows, false, 0, A.at<QBlock>(ap.o_qb), ap.n_qb, fin);
    }
    // order every admission write (page table, target lengths, prompts, actor
    // KV) before the next decode on sa and the next scorer wave on ss, also
    // when no prefill pass ran (all prompts of length 1)
    OPPO_CUDA_CHECK(cudaEventRecord(e.ev_admit, st));
    for (cudaStream_t o : {e.sa, e.ss})
        if (o != st) OPPO_CUDA_CHECK(cudaStreamWaitEvent(o, e.ev_admit, 0));
}

}  // namespace

// ================================================================ run_step
namespace {

struct PassPlan {
    size_t seg_off = 0, qb_off = 0, lm_off = 0, pend_off = 0;
    int n_seg = 0, n_qb = 0, rows = 0, n_lm = 0, n_pend = 0;
};
struct WavePlan {
    int at_iter = 0;  // 0 = before decode
    std::vector<PassPlan> passes;
};

struct SegReq {
    int slot, pos0, n, prompt_len;
};

// Splits a wave's segments into passes of <= cap rows and builds the
// reference-model lm_head rows (pending resolution) for each pass.
void build_passes(Engine& e, std::vector<SegReq>& reqs, WavePlan& wave, Arena& A) {
    const int cap = e.ws.max_rows;
    size_t i = 0;
    int off_in_seg = 0;
    while (i < reqs.size()) {
        std::vector<Segment> segs;
        std::vector<QBlock> qbs;
        std::vector<LmRow> lms;
        std::vector<int32_t> psrc, pslot;
        int rows = 0;
        while (i < reqs.size() && rows < cap) {
            const SegReq& r = reqs[i];
            const int take = std::min(r.n - off_in_seg, cap - rows);
            const int pos0 = r.pos0 + off_in_seg;
            segs.push_back({r.slot, pos0, take, rows, r.prompt_len, 0});
            for (int b = 0; b < take; b += e.qblock)
                qbs.push_back({rows + b, std::min(e.qblock, take - b), r.slot, pos0 + b});
            auto& info = e.slots[r.slot];
            const int P = r.prompt_len, L = info.target_len;
            // resolve this slot's pending reference row: its target is the token at pos0
            if (info.ref_pending) {
                lms.push_back({-(r.slot + 1), r.slot, pos0 - P + 1, 0});
                info.ref_pending = false;
            }
            for (int k = 0; k < take; ++k) {
                const int q = pos0 + k, t = q - P + 2;  // target response index of row q
                if (t < 1 || t > L) continue;
                if (k + 1 < take) {
                    lms.push_back({rows + k, r.slot, t, 0});
                } else {  // target not in this pass yet
                    psrc.push_back(rows + k);
                    pslot.push_back(r.slot);
                    info.ref_pending = true;
                }
            }
            rows += take;
            off_in_seg += take;
            if (off_in_seg >= r.n) {
                ++i;
                off_in_seg = 0;
            }
        }
        PassPlan p;
        p.seg_off = A.push_vec(segs);
        p.n_seg = static_cast<int>(segs.size());
        p.qb_off = A.push_vec(qbs);
        p.n_qb = static_cast<int>(qbs.size());
        p.lm_off = A.push_vec(lms);
        p.n_lm = static_cast<int>(lms.size());
        std::vector<int32_t> pend(psrc);  // [src rows | slots], one contiguous block
        pend.insert(pend.end(), pslot.begin(), pslot.end());
        p.pend_off = A.push_vec(pend);
        p.n_pend = static_cast<int>(psrc.size());
        p.rows = rows;
        wave.passes.push_back(p);
    }
}

template <class T>
void run_scorer_pass(Engine& e, const PassPlan& p, Arena& A, cudaStream_t st, int64_t& tokens) {
    Work& w = e.ws;
    segment_rows<<<p.n_seg, 128, 0, st>>>(A.at<Segment>(p.seg_off), e.d_prompt, e.Pmax, e.d_tok,
                                          e.tok_stride, w.meta);
    const QBlock* qb = A.at<QBlock>(p.qb_off);
    tokens += p.rows;
    // three concurrent model passes: critic and reference on their own
    // streams / workspaces (row metadata shared), joined before the next
    // pass rewrites the metadata
    const bool conc = e.scorer_streams == 3;
    Work wc = conc ? e.ws_m[0] : w, wr = conc ? e.ws_m[1] : w;
    cudaStream_t sc = st, sr = st;
    if (conc) {
        wc.meta = w.meta;
        wr.meta = w.meta;
        sc = e.ss_m[0];
        sr = e.ss_m[1];
        OPPO_CUDA_CHECK(cudaEventRecord(e.ev_seg, st));
        OPPO_CUDA_CHECK(cudaStreamWaitEvent(sc, e.ev_seg, 0));
        OPPO_CUDA_CHECK(cudaStreamWaitEvent(sr, e.ev_seg, 0));
    }
    // reward model: last-token scalar head
    {
        Final<T> fin;
        fin.write_h = false;
        fin.head = e.models[REWARD].head;
        forward<T>(e, e.models[REWARD], w, st, p.rows, false, 0, qb, p.n_qb, fin);
        reward_rows<<<cdiv(p.rows, 256), 256, 0, st>>>(w.head_out, w.meta.slot, w.meta.t, p.rows,
                                                       e.d_target_len, e.d_reward);
    }
    // critic: per-token value head (state before token t) + hidden cache for the head update
    {
        Final<T> fin;
        fin.write_h = false;
        fin.head = e.models[CRITIC].head;
        fin.cache = static_cast<T*>(e.d_hf_critic);
        fin.t_lo = 1;
        fin.t_hi = e.Lmax;
        forward<T>(e, e.models[CRITIC], wc, sc, p.rows, false, 0, qb, p.n_qb, fin);
        scatter_rows<<<cdiv(p.rows, 256), 256, 0, sc>>>(wc.head_out, wc.meta.slot, wc.meta.t, p.rows,
                                                        e.d_values, e.tok_stride, 1, e.d_target_len, 0);
    }
    // reference: log-probs of the actor's tokens (lm_head + log-sum-exp)
    {
        Model& m = e.models[REF];
        Final<T> fin;
        fin.write_h = true;
        forward<T>(e, m, wr, sr, p.rows, false, 0, qb, p.n_qb, fin);
        const int D = m.dims.d_model;
        if (p.n_lm > 0) {
            gather_lm_rows<T><<<p.n_lm, 128, 0, sr>>>(A.at<LmRow>(p.lm_off), p.n_lm,
                                                      static_cast<const T*>(wr.h),
                                                      static_cast<const T*>(e.d_ref_pending), D,
                                                      e.d_tok, e.tok_stride, static_cast<T*>(wr.lm_in),
                                                      wr.lm_tgt, wr.lm_slot, wr.lm_t);
            EpiParams ep{};
            ep.mode = EPI_LOGITS;
            ep.partials = wr.partials;
            ep.tgt_logit = wr.tgt_logit;
            ep.targets = wr.lm_tgt;
            ep.keys = nullptr;
            gemm_run(e, wr, sr, wr.lm_in, p.n_lm, D, D, m.lm_head, m.dims.vocab, D, ep);
            logits_combine<<<cdiv(p.n_lm, 4), 128, 0, sr>>>(
                wr.partials, gemm_logit_tiles(e.dtype, m.dims.vocab), m.dims.vocab, p.n_lm, nullptr, wr.tgt_logit, wr.lm_slot, wr.lm_t,
                nullptr, e.d_ref_lp, e.tok_stride, nullptr, nullptr);
        }
        if (p.n_pend > 0)
            store_pending<T><<<p.n_pend, 128, 0, sr>>>(A.at<int32_t>(p.pend_off),
                                                       A.at<int32_t>(p.pend_off) + p.n_pend, p.n_pend,
                                                       static_cast<const T*>(wr.h),
                                                       static_cast<T*>(e.d_ref_pending), D);
    }
    if (conc) {  // the next pass's segment_rows rewrites the shared metadata
        OPPO_CUDA_CHECK(cudaEventRecord(e.ev_m[0], sc));
        OPPO_CUDA_CHECK(cudaEventRecord(e.ev_m[1], sr));
        OPPO_CUDA_CHECK(cudaStreamWaitEvent(st, e.ev_m[0], 0));
        OPPO_CUDA_CHECK(cudaStreamWaitEvent(st, e.ev_m[1], 0));
    }
    e.launches += 8;
    OPPO_CUDA_CHECK(cudaGetLastError());
}

// Rows [0, M) of one decode iteration through `w` (meta already filled):
// forward, lm_head + in-block sampling, combine (token, log-prob -> buffers).
template <class T>
void decode_rows_forward(Engine& e, Work& w, int M, cudaStream_t st, int32_t* iter_inc) {
    Model& m = e.models[ACTOR];
    const int max_ctx = e.Pmax + e.Lmax;
    Final<T> fin;
    fin.write_h = true;
    fin.cache = static_cast<T*>(e.d_hf_actor);
    fin.t_lo = 1;
    fin.t_hi = e.Lmax;
    forward<T>(e, m, w, st, M, true, max_ctx, nullptr, 0, fin);
    EpiParams ep{};
    ep.mode = EPI_LOGITS;
    ep.partials = w.partials;
    ep.tgt_logit = w.tgt_logit;
    ep.targets = nullptr;
    ep.keys = w.meta.key;
    const int D = m.dims.d_model;
    if (std::is_same_v<T, __nv_bfloat16> && M <= e.lmhead_dec_max && D % 64 == 0 && m.dims.vocab % 128 == 0)
        lmhead_dec_run(e, w, st, w.h, M, D, m.lm_head, m.dims.vocab, w.partials, w.meta.key);
    else
        gemm_run(e, w, st, w.h, M, D, D, m.lm_head, m.dims.vocab, D, ep);
    launch(e.pdl, logits_combine, dim3(cdiv(M, 4)), dim3(128), 0, st, w.partials, gemm_logit_tiles(e.dtype, m.dims.vocab), m.dims.vocab, M, w.meta.key,
                                               nullptr, w.meta.slot, w.meta.t, e.d_tok, e.d_old_lp,
                                               e.tok_stride, nullptr, nullptr, iter_inc);
    e.launches += 2;
}

template <class T>
void decode_iteration(Engine& e, int M, cudaStream_t st) {
    Work& w = e.wa;
    launch(e.pdl, decode_rows, dim3(cdiv(M, 128)), dim3(128), 0, st, e.d_dseq, M, e.d_iter, e.d_prompt, e.Pmax, e.d_tok,
                                              e.tok_stride, e.cfg.sample_seed, w.meta, e.S);
    e.launches += 1;
    if (e.dec_split_min > 0 && M >= e.dec_split_min && M >= 32) {
        // two concurrent halves: rows [0, M1) on st through wa, [M1, M) on sa2
        // through wa2 viewing wa's row metadata; the iteration counter is
        // advanced by the second half only (both read it in decode_rows above)
        const int M1 = (M / 2 + 15) / 16 * 16;
        static const int pct = env_int("OPPO_DEC_SPLIT_SMS_PCT", 50);  // grid sizing per half (measured best)
        Work wa_h = w;
        wa_h.sms = std::max(8, w.sms * pct / 100);
        Work wb = e.wa2;
        wb.sms = wa_h.sms;
        wb.meta.slot = w.meta.slot + M1;
        wb.meta.pos = w.meta.pos + M1;
        wb.meta.tok = w.meta.tok + M1;
        wb.meta.t = w.meta.t + M1;
        wb.meta.key = w.meta.key + M1;
        OPPO_CUDA_CHECK(cudaEventRecord(e.ev_fork, st));
        OPPO_CUDA_CHECK(cudaStreamWaitEvent(e.sa2, e.ev_fork, 0));
        decode_rows_forward<T>(e, wb, M - M1, e.sa2, e.d_iter);
        decode_rows_forward<T>(e, wa_h, M1, st, nullptr);
        OPPO_CUDA_CHECK(cudaEventRecord(e.ev_join, e.sa2));
        OPPO_CUDA_CHECK(cudaStreamWaitEvent(st, e.ev_join, 0));
    } else {
        decode_rows_forward<T>(e, w, M, st, e.d_iter);
    }
}

// One decode iteration for batch size M: replay the captured graph (capture on
// first use).  Host cost per iteration is one cudaGraphLaunch.
template <class T>
cudaGraphExec_t ensure_decode_graph(Engine& e, int M, cudaStream_t st, bool long_ctx) {
    const int key = 2 * M + (long_ctx ? 1 : 0);  // two variants per bucket: split-KV attention or not
    auto it = e.decode_graphs.find(key);
    if (it == e.decode_graphs.end()) {
        const int64_t before = e.launches;
        cudaGraph_t g;
        e.attn_long = long_ctx;
        OPPO_CUDA_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
            decode_iteration<T>(e, M, st);
        } catch (...) {
            cudaStreamEndCapture(st, &g);
            e.attn_long = false;
            throw;
        }
        e.attn_long = false;
        OPPO_CUDA_CHECK(cudaStreamEndCapture(st, &g));
        cudaGraphExec_t ge;
        OPPO_CUDA_CHECK(cudaGraphInstantiate(&ge, g, 0));
        OPPO_CUDA_CHECK(cudaGraphDestroy(g));
        OPPO_CUDA_CHECK(cudaGraphUpload(ge, st));  // device-side setup now, not at the first launch
        it = e.decode_graphs.emplace(key, ge).first;
        e.decode_graph_launches[key] = e.launches - before;
        e.launches = before;
    }
    return it->second;
}

template <class T>
void decode_iteration_graph(Engine& e, int M, cudaStream_t st, bool long_ctx) {
    if (!e.cfg.use_graphs) {
        e.attn_long = long_ctx;
        decode_iteration<T>(e, M, st);
        e.attn_long = false;
        return;
    }
    OPPO_CUDA_CHECK(cudaGraphLaunch(ensure_decode_graph<T>(e, M, st, long_ctx), st));
    e.launches += e.decode_graph_launches[2 * M + (long_ctx ? 1 : 0)];
}

// ------------------------------------ policy log-probs of the finished sequences
// meta = [n slots][n + 1 token offsets]
template <class T>
__global__ void pre_gather(const int32_t* __restrict__ meta, int n, const int32_t* __restrict__ tok,
                           const T* __restrict__ cache, int stride, int d, int32_t* o_tok, T* o_hf) {
    const int i = blockIdx.y;
    const int s = meta[i], a = meta[n + i], L = meta[n + i + 1] - a;
    for (int t = blockIdx.x; t < L; t += gridDim.x) {
        const size_t src = static_cast<size_t>(s) * stride + t + 1;
        if (threadIdx.x == 0) o_tok[a + t] = tok[src];
        const T* h = cache + src * d;
        T* dst = o_hf + static_cast<size_t>(a + t) * d;
        for (int k = threadIdx.x; k < d; k += blockDim.x) dst[k] = h[k];
    }
}

// log pi(token) and the log-sum-exp of every sampled token of the sequences
// that finished this step, under the current lm_head, on stream `st` (the
// actor's SMs, idle while the scorers finish the last wave).  Same kernels,
// tiles and per-row arithmetic as the recompute in ppo_update_impl (a
// LOGITS row never depends on the other rows of its tile), so the update
// that reuses them is bit-identical to one that recomputes.
template <class T>
void precompute_policy_lp(Engine& e, const std::vector<int>& fslots, cudaStream_t st) {
    e.pre_index.clear();
    e.pre_version = -1;
    const int n = static_cast<int>(fslots.size());
    if (n == 0) return;
    Model& actor = e.models[ACTOR];
    const int Da = actor.dims.d_model, V = actor.dims.vocab;
    std::vector<int32_t> meta(2 * n + 1);
    int N = 0;
    for (int i = 0; i < n; ++i) {
        const auto& info = e.slots[fslots[i]];
        meta[i] = fslots[i];
        meta[n + i] = N;
        e.pre_index[info.id] = {N, info.target_len};
        N += info.target_len;
    }
    meta[2 * n] = N;
    if (N == 0) return;
    if (static_cast<size_t>(N) > e.pre_cap) {
        for (void* p : {e.pre_hf, static_cast<void*>(e.pre_tok), static_cast<void*>(e.pre_new),
                        static_cast<void*>(e.pre_lse)})
            if (p) cudaFree(p);
        e.pre_cap = static_cast<size_t>(N) * 5 / 4 + 64;
        e.pre_hf = dalloc(e.pre_cap * Da * e.esz);
        e.pre_tok = static_cast<int32_t*>(dalloc(e.pre_cap * 4));
        e.pre_new = static_cast<float*>(dalloc(e.pre_cap * 4));
        e.pre_lse = static_cast<float*>(dalloc(e.pre_cap * 4));
    }
    if (2 * n + 1 > e.pre_meta_cap) {
        if (e.pre_meta) cudaFree(e.pre_meta);
        e.pre_meta_cap = 2 * n + 65;
        e.pre_meta = static_cast<int32_t*>(dalloc(static_cast<size_t>(e.pre_meta_cap) * 4));
    }
    const int nt = gemm_logit_tiles(e.dtype, V);
    if (!e.pre_partials) {
        e.pre_chunk = std::max(128, std::min(8192, static_cast<int>((static_cast<size_t>(64) << 20) / (nt * 16))));
        e.pre_partials = static_cast<float4*>(dalloc(static_cast<size_t>(e.pre_chunk) * nt * 16));
        e.pre_tgt = static_cast<float*>(dalloc(static_cast<size_t>(e.pre_chunk) * 4));
    }
    OPPO_CUDA_CHECK(cudaMemcpyAsync(e.pre_meta, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice, st));
    pre_gather<T><<<dim3(64, n), 128, 0, st>>>(e.pre_meta, n, e.d_tok, static_cast<const T*>(e.d_hf_actor),
                                               e.tok_stride, Da, e.pre_tok, static_cast<T*>(e.pre_hf));
    for (int c0 = 0; c0 < N; c0 += e.pre_chunk) {
        const int cn = std::min(e.pre_chunk, N - c0);
        EpiParams ep{};
        ep.mode = EPI_LOGITS;
        ep.partials = e.pre_partials;
        ep.tgt_logit = e.pre_tgt;
        ep.targets = e.pre_tok + c0;
        gemm_run(e, e.wa, st, static_cast<const T*>(e.pre_hf) + static_cast<size_t>(c0) * Da, cn, Da, Da,
                 actor.lm_head, V, Da, ep);
        logits_combine<<<cdiv(cn, 4), 128, 0, st>>>(e.pre_partials, nt, V, cn, nullptr, e.pre_tgt, nullptr, nullptr,
                                                    nullptr, e.pre_new + c0, 0, e.pre_lse + c0, nullptr);
    }
    e.launches += 1 + 2 * cdiv(N, e.pre_chunk);
    OPPO_CUDA_CHECK(cudaGetLastError());
    OPPO_CUDA_CHECK(cudaEventRecord(e.ev_pre, st));
    e.pre_version = e.lm_version;
}

template <class T>
void run_step_impl(Engine& e, const std::vector<oppo_seq_state>& active, int chunk, int mode,
                   int stop_after, std::vector<oppo_seq_outcome>& out, oppo_ledger& ledger) {
    const StepPlan plan = plan_step(active, chunk, mode, stop_after, e.cfg.carry_granularity);
    open_step(e);
    const int n = static_cast<int>(active.size());
    const int64_t t_end = plan.t_end;
    std::vector<int> slot(n);
    for (int i = 0; i < n; ++i) {
        auto it = e.slot_of.find(active[i].id);
        if (it == e.slot_of.end()) input_error("sequence " + std::to_string(active[i].id) + " not admitted");
        slot[i] = it->second;
        if (e.slots[slot[i]].target_len != active[i].target_len)
            input_error("target_len changed since admission");
    }
    // decode order: remaining length descending, so the batch of iteration t is a prefix
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        const int ra = active[a].target_len - active[a].generated;
        const int rb = active[b].target_len - active[b].generated;
        return ra != rb ? ra > rb : active[a].id < active[b].id;
    });
    std::vector<DecodeSeq> dseq;
    std::vector<int> rem_sorted;
    for (int i : order) {
        const int rem = active[i].target_len - active[i].generated;
        if (rem <= 0) continue;
        dseq.push_back({slot[i], active[i].prompt_len, active[i].generated, active[i].target_len,
                        active[i].id});
        rem_sorted.push_back(rem);
    }
    auto& A = g_extra[&e].step_arena;
    A.host.clear();
    const size_t n_dec = dseq.size();
    while (static_cast<int>(dseq.size()) < e.S + 16)  // padding rows -> scratch slot on device
        dseq.push_back({e.S, 1, 0, -1, -1});
    const size_t o_dseq = A.push_vec(dseq);

    // ---------------------------------------------------------- wave plans
    const bool streamed = mode == OPPO_MODE_STREAMED;
    std::vector<int> p_cur(n);
    for (int i = 0; i < n; ++i) p_cur[i] = active[i].prefilled_tokens;
    std::vector<WavePlan> waves;
    int64_t wave_tokens = 0;
    double pf_flops = 0, pf_bytes = 0, scorer_params[N_MODELS] = {0}, kv_bytes_tok[N_MODELS] = {0};
    for (int mi : {REWARD, CRITIC, REF}) {  // non-embedding parameters; K+V bytes per token
        const auto& d = e.models[mi].dims;
        scorer_params[mi] = static_cast<double>(d.n_layers) *
            ((static_cast<double>(d.n_heads + 2 * d.n_kv_heads) * d.head_dim + d.n_heads * d.head_dim) * d.d_model +
             3.0 * d.d_model * d.d_ff);
        kv_bytes_tok[mi] = 2.0 * d.n_layers * d.n_kv_heads * d.head_dim * e.esz;
    }
    // Streamed mode scores the prompts of fresh sequences in the wave at tick 0
    // (the scorer partition is otherwise idle until the first chunk is decoded);
    // their first response chunk then starts at position P.  Decisions do not
    // change (prefill time is 0 on the logical clock); numerics are per row.
    const bool prompts_at_0 = streamed && e.prompt_t0;
    auto make_wave = [&](int at_iter, auto&& target_p) {
        std::vector<SegReq> reqs;
        for (int i : order) {  // deterministic order
            const int want = target_p(i);
            if (want <= p_cur[i]) {
                auto& inf = e.slots[slot[i]];
                if (at_iter == 0 && prompts_at_0 && p_cur[i] == 0 && !inf.scored_prompt) {
                    const int P = active[i].prompt_len;
                    reqs.push_back({slot[i], 0, P, P});  // prompt only: positions 0 .. P-1
                    inf.scored_prompt = true;
                }
                continue;
            }
            auto& info = e.slots[slot[i]];
            const int P = active[i].prompt_len;
            const bool first = p_cur[i] == 0 && !info.scored_prompt;
            const int pos0 = first ? 0 : P + p_cur[i];
            const int pos1 = P + want - 1;
            reqs.push_back({slot[i], pos0, pos1 - pos0 + 1, P});
            info.scored_prompt = true;
            p_cur[i] = want;
        }
        if (reqs.empty()) return;
        WavePlan wv;
        wv.at_iter = at_iter;
        build_passes(e, reqs, wv, A);
        // algorithmic work of the wave (SURVEY 8d F_pf / B_pf)
        for (const auto& r : reqs) {
            const double n = r.n, ctx = n * r.pos0 + n * (n + 1) / 2;  // sum of causal context lengths
            const double resp = std::max(0, r.pos0 + r.n - std::max(r.pos0, r.prompt_len));  // ref lm_head rows
            for (int mi : {REWARD, CRITIC, REF}) {
                const auto& d = e.models[mi].dims;
                pf_flops += 2.0 * scorer_params[mi] * n + 4.0 * d.n_layers * d.n_heads * d.head_dim * ctx;
                pf_bytes += kv_bytes_tok[mi] * (n + r.pos0 + n);  // append n rows, read the context once
            }
            pf_flops += 2.0 * e.models[REF].dims.vocab * e.models[REF].dims.d_model * resp;
        }
        for (size_t k = 0; k < wv.passes.size(); ++k)
            for (int mi : {REWARD, CRITIC, REF}) pf_bytes += scorer_params[mi] * e.esz;
        pf_bytes += e.esz * static_cast<double>(e.models[REF].dims.vocab) * e.models[REF].dims.d_model *
                    wv.passes.size();  // the reference model's lm_head per pass
        waves.push_back(std::move(wv));
    };
    auto whole_by = [&](int i, int64_t t) -> int {  // chunk-complete tokens after iteration t
        const auto& s = active[i];
        const int64_t rem = s.target_len - s.generated;
        const int64_t rel = rem <= t ? rem : (t / chunk) * chunk;
        return static_cast<int>(s.generated + rel);
    };
    if (streamed) {
        make_wave(0, [&](int i) { return active[i].generated; });  // carried chunks, at tick 0
        for (int64_t t = chunk; t < t_end; t += chunk)
            make_wave(static_cast<int>(t), [&](int i) { return whole_by(i, t); });
        make_wave(static_cast<int>(t_end), [&](int i) { return whole_by(i, t_end); });
    } else {
        make_wave(static_cast<int>(t_end), [&](int i) {
            const auto& s = active[i];
            const int64_t rem = s.target_len - s.generated;
            return rem <= t_end ? s.target_len : s.generated;
        });
    }
    // sanity: the prefilled counts must equal the logical outcome's
    for (int i = 0; i < n; ++i) {
        const int expect = active[i].prefilled_tokens + plan.outcomes[i].tokens_prefilled;
        if (p_cur[i] != expect)
            internal_error("wave plan disagrees with the logical clock (seq " +
                           std::to_string(active[i].id) + ")");
    }
    A.upload(e.sa);
    OPPO_CUDA_CHECK(cudaMemcpyAsync(e.d_dseq, A.at<DecodeSeq>(o_dseq), dseq.size() * sizeof(DecodeSeq),
                                    cudaMemcpyDeviceToDevice, e.sa));
    set_int<<<1, 1, 0, e.sa>>>(e.d_iter, 1);

    // ------------------------------------------------------------- enqueue
    while (e.ev_wave.size() < 2 * waves.size()) {
        cudaEvent_t ev;
        OPPO_CUDA_CHECK(cudaEventCreate(&ev));
        e.ev_wave.push_back(ev);
    }
    if (e.ev_pool.size() < waves.size() + 2) {
        const size_t old = e.ev_pool.size();
        e.ev_pool.resize(waves.size() + 2);
        for (size_t i = old; i < e.ev_pool.size(); ++i)
            OPPO_CUDA_CHECK(cudaEventCreateWithFlags(&e.ev_pool[i], cudaEventDisableTiming));
    }
    OPPO_CUDA_CHECK(cudaStreamWaitEvent(e.ss, e.ev_begin, 0));
    // the scorer stream must also see the arena upload and admission prefill on sa
    OPPO_CUDA_CHECK(cudaEventRecord(e.ev_pool[0], e.sa));
    OPPO_CUDA_CHECK(cudaStreamWaitEvent(e.ss, e.ev_pool[0], 0));
    size_t wi = 0;
    int64_t decode_tokens = 0;
    std::atomic<int64_t> prefill_tokens{0};
    ScorerWorker& worker = g_extra[&e].scorer;
    worker.start(e.cfg.device);
    struct DrainOnUnwind {  // posted jobs reference this frame: never leave it with jobs queued
        ScorerWorker& w;
        ~DrainOnUnwind() {
            try {
                w.drain();
            } catch (...) {
            }
        }
    } drain_guard{worker};
    const bool flags = e.chunk_flags;
    if (flags && e.cfg.use_graphs) {
        // every decode graph this step can launch exists (captured, instantiated,
        // uploaded) before a scorer kernel starts polling: first-time setup of a
        // graph or kernel must not wait behind a spinning poller
        const int top = std::min(cdiv(static_cast<int64_t>(n_dec), 16) * 16, e.S + 16);
        bool any_long = false;  // can an iteration of this step reach the long-context variant
        for (size_t r = 0; r < n_dec; ++r)
            any_long |= dseq[r].prompt_len + dseq[r].target_len >= e.attn_long_ctx;
        for (int bkt = 16; bkt <= top; bkt += 16) {
            ensure_decode_graph<T>(e, bkt, e.sa, false);
            if (any_long && e.attn_max_split != 1) ensure_decode_graph<T>(e, bkt, e.sa, true);
        }
    }
    std::vector<uint32_t> wave_seq(waves.size());
    for (size_t k = 0; flags && k < waves.size(); ++k) wave_seq[k] = ++e.ready_seq;
    // With flags the scorer stream's copy of wave k is enqueued one wave ahead
    // (when wave k-1's flag is written), gated on the device by wave k's flag.
    auto post_wave = [&](size_t k) {
        const uint32_t* flag = e.d_ready + (wave_seq[k] % Engine::kReadyRing);
        const uint32_t want = wave_seq[k];
        const WavePlan* wave = &waves[k];
        cudaEvent_t t0 = e.ev_wave[2 * k], t1 = e.ev_wave[2 * k + 1];
        worker.post([&e, &A, &prefill_tokens, flag, want, wave, t0, t1] {
            wait_ready<<<1, 32, 0, e.ss>>>(flag, want);
            OPPO_CUDA_CHECK(cudaGetLastError());
            e.launches += 1;
            OPPO_CUDA_CHECK(cudaEventRecord(t0, e.ss));  // the wave's chunks are ready
            int64_t tok = 0;
            for (const auto& p : wave->passes) run_scorer_pass<T>(e, p, A, e.ss, tok);
            OPPO_CUDA_CHECK(cudaEventRecord(t1, e.ss));
            prefill_tokens += tok;
        });
    };
    if (flags && !waves.empty()) post_wave(0);
    auto fire_waves_at = [&](int64_t it) {
        while (wi < waves.size() && waves[wi].at_iter == it) {
            if (flags) {  // actor-stream order: after iteration `it`, the wave's chunks are complete
                set_ready<<<1, 32, 0, e.sa>>>(e.d_ready + (wave_seq[wi] % Engine::kReadyRing), wave_seq[wi]);
                OPPO_CUDA_CHECK(cudaGetLastError());
                e.launches += 1;
                if (wi + 1 < waves.size()) post_wave(wi + 1);
                ++wi;
                continue;
            }
            cudaEvent_t ev = e.ev_pool[wi + 1];
            OPPO_CUDA_CHECK(cudaEventRecord(ev, e.sa));  // actor-stream order: after iteration `it`
            const WavePlan* wave = &waves[wi];
            cudaEvent_t t0 = e.ev_wave[2 * wi], t1 = e.ev_wave[2 * wi + 1];
            worker.post([&e, &A, &prefill_tokens, ev, wave, t0, t1] {
                OPPO_CUDA_CHECK(cudaStreamWaitEvent(e.ss, ev, 0));
                OPPO_CUDA_CHECK(cudaEventRecord(t0, e.ss));  // the wave's chunks are ready
                int64_t tok = 0;
                for (const auto& p : wave->passes) run_scorer_pass<T>(e, p, A, e.ss, tok);
                OPPO_CUDA_CHECK(cudaEventRecord(t1, e.ss));  // (passes end joined back on ss)
                prefill_tokens += tok;
            });
            ++wi;
        }
    };
    fire_waves_at(0);
    const auto host_t0 = std::chrono::steady_clock::now();
    size_t active_n = n_dec;
    // algorithmic bytes of the decode loop: weights once per
    // iteration + per active row the KV it reads (ctx positions) and appends
    const auto& ad = e.models[ACTOR].dims;
    const double w_bytes = static_cast<double>(e.esz) *
        (static_cast<double>(ad.n_layers) *
             ((static_cast<double>(ad.n_heads + 2 * ad.n_kv_heads) * ad.head_dim + ad.n_heads * ad.head_dim) *
                  ad.d_model +
              3.0 * ad.d_model * ad.d_ff) +
         static_cast<double>(ad.vocab) * ad.d_model);
    const double kvb = 2.0 * ad.n_layers * ad.n_kv_heads * ad.head_dim * e.esz;  // K+V per token
    double loop_w = 0, loop_kv = 0, loop_f = 0;
    const double p_dec = w_bytes / e.esz;  // non-embedding + lm_head parameters
    const double att_f = 4.0 * ad.n_layers * ad.n_heads * ad.head_dim;  // per (token, context position)
    OPPO_CUDA_CHECK(cudaEventRecord(e.ev_loop0, e.sa));
    for (int64_t it = 1; it <= t_end; ++it) {
        while (active_n > 0 && rem_sorted[active_n - 1] < it) --active_n;
        if (active_n == 0) break;
        loop_w += w_bytes;
        int64_t ctx_max = 0;
        for (size_t r = 0; r < active_n; ++r) {
            const DecodeSeq& q = dseq[r];
            const int64_t ctx = q.prompt_len + q.generated + it;
            loop_kv += kvb * static_cast<double>(ctx);  // ctx + appended row
            loop_f += 2.0 * p_dec + att_f * static_cast<double>(ctx);
            ctx_max = std::max(ctx_max, ctx);
        }
        // long-context iteration: split-KV decode attention (graph variant)
        const bool long_ctx = e.attn_max_split != 1 && ctx_max >= e.attn_long_ctx;
        // bucketed batch: rows [active_n, bucket) decode into the scratch slot
        const int bucket = e.cfg.use_graphs ? std::min(cdiv(active_n, 16) * 16, e.S + 16)
                                            : static_cast<int>(active_n);
        decode_iteration_graph<T>(e, bucket, e.sa, long_ctx);
        decode_tokens += static_cast<int64_t>(active_n);
        if (it == t_end) OPPO_CUDA_CHECK(cudaEventRecord(e.ev_dec_end, e.sa));
        fire_waves_at(it);
    }
    if (active_n == 0 || t_end == 0) OPPO_CUDA_CHECK(cudaEventRecord(e.ev_dec_end, e.sa));
    const double host_enqueue_us =
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - host_t0).count();
    if (std::getenv("OPPO_DEBUG_TIMING"))
        std::fprintf(stderr, "[oppo] decode enqueue host %.1f ms for %lld iterations, tma maps %zu\n",
                     host_enqueue_us / 1e3, static_cast<long long>(t_end), e.tma_cache.size());
    fire_waves_at(t_end);  // (t_end == 0 or already fired: no-op)
    if (wi != waves.size()) internal_error("unfired scorer waves");
    if (e.pre_lp) {  // the actor SMs are idle until the scorers finish: policy log-probs for the update
        std::vector<int> fs;
        for (int i = 0; i < n; ++i)
            if (active[i].generated + plan.outcomes[i].tokens_decoded >= active[i].target_len) fs.push_back(slot[i]);
        precompute_policy_lp<T>(e, fs, e.sa);
    }
    worker.drain();  // every scorer launch is enqueued on ss (rethrows a worker error)
    OPPO_CUDA_CHECK(cudaEventRecord(e.ev_sc_end, e.ss));
    OPPO_CUDA_CHECK(cudaStreamWaitEvent(e.sa, e.ev_sc_end, 0));
    OPPO_CUDA_CHECK(cudaEventRecord(e.ev_done, e.sa));
    OPPO_CUDA_CHECK(cudaEventSynchronize(e.ev_done));
    OPPO_CUDA_CHECK(cudaGetLastError());
    e.step_open = false;

    out = plan.outcomes;
    ledger = plan.ledger;
    float ms = 0;
    OPPO_CUDA_CHECK(cudaEventElapsedTime(&ms, e.ev_begin, e.ev_done));
    ledger.step_us = ms * 1e3;
    OPPO_CUDA_CHECK(cudaEventElapsedTime(&ms, e.ev_begin, e.ev_dec_end));
    ledger.decode_us = ms * 1e3;
    OPPO_CUDA_CHECK(cudaEventElapsedTime(&ms, e.ev_begin, e.ev_sc_end));
    ledger.score_us = ms * 1e3;
    double busy = 0;  // scorer partition busy time: sum of the waves' spans
    for (size_t k = 0; k < waves.size(); ++k) {
        OPPO_CUDA_CHECK(cudaEventElapsedTime(&ms, e.ev_wave[2 * k], e.ev_wave[2 * k + 1]));
        busy += ms * 1e3;
    }
    ledger.score_busy_us = busy;
    OPPO_CUDA_CHECK(cudaEventElapsedTime(&ms, e.ev_loop0, e.ev_dec_end));
    ledger.decode_loop_us = ms * 1e3;
    ledger.decode_weight_bytes = loop_w;
    ledger.decode_kv_bytes = loop_kv;
    ledger.decode_flops = loop_f;
    ledger.prefill_flops = pf_flops;
    ledger.prefill_bytes = pf_bytes;
    ledger.decode_iters = t_end;
    ledger.decode_tokens = decode_tokens;
    ledger.prefill_tokens = prefill_tokens;
    ledger.kernel_launches = e.launches;
}

// =============================================================== PPO update
template <class T>
__global__ void gather_batch(const int32_t* __restrict__ slots, const int32_t* __restrict__ off,
                             int n, const int32_t* __restrict__ tok, const float* __restrict__ old_lp,
                             const float* __restrict__ ref_lp, const float* __restrict__ vals,
                             const float* __restrict__ reward, int stride, int32_t* o_tok,
                             float* o_old, float* o_ref, float* o_vtok, float* o_vals,
                             float* o_score) {
    const int i = blockIdx.x;
    if (i >= n) return;
    const int s = slots[i], a = off[i], L = off[i + 1] - a;
    for (int t = threadIdx.x; t < L; t += blockDim.x) {
        const size_t src = static_cast<size_t>(s) * stride + t + 1;
        o_tok[a + t] = tok[src];
        o_old[a + t] = old_lp[src];
        o_ref[a + t] = ref_lp[src];
        o_vtok[a + t] = vals[src];
        o_vals[a + i + t] = vals[src];
    }
    if (threadIdx.x == 0) {
        o_vals[a + i + L] = 0.f;  // terminal convention (ppo.cpp:278)
        o_score[i] = reward[s];
    }
}
__global__ void gather_pre_lp(const int32_t* __restrict__ src, const int32_t* __restrict__ off, int n,
                              const float* __restrict__ pre_new, const float* __restrict__ pre_lse, float* o_new,
                              float* o_lse) {
    const int i = blockIdx.x;
    if (i >= n) return;
    const int a = off[i], L = off[i + 1] - a, b = src[i];
    for (int t = threadIdx.x; t < L; t += blockDim.x) {
        o_new[a + t] = pre_new[b + t];
        o_lse[a + t] = pre_lse[b + t];
    }
}
template <class T>
__global__ void gather_hidden(const int32_t* __restrict__ slots, const int32_t* __restrict__ off,
                              int n, const T* __restrict__ cache, int stride, int d, T* out) {
    const int i = blockIdx.y;
    const int s = slots[i], a = off[i], L = off[i + 1] - a;
    for (int t = blockIdx.x; t < L; t += gridDim.x) {
        const T* src = cache + (static_cast<size_t>(s) * stride + t + 1) * d;
        T* dst = out + static_cast<size_t>(a + t) * d;
        for (int k = threadIdx.x; k < d; k += blockDim.x) dst[k] = src[k];
    }
}
template <class T>
__global__ void transpose_rows(const T* __restrict__ in, int rows, int cols, int ld_out, T* out) {
    __shared__ T tile[32][33];
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        tile[i][threadIdx.x] = (r < rows && c < cols) ? in[static_cast<size_t>(r) * cols + c] : fromf<T>(0.f);
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, r = r0 + threadIdx.x;
        if (c < cols && r < ld_out) out[static_cast<size_t>(c) * ld_out + r] = tile[threadIdx.x][i];
    }
}
__global__ void sum_partials(const double* p, int n, double* out) {
    if (threadIdx.x) return;
    double s = 0;
    for (int i = 0; i < n; ++i) s += p[i];
    out[0] = s;
}
__global__ void head_sgd(float* w, const float* g, int d, float lr) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < d) w[i] -= lr * g[i];
}
__global__ void sq_err_sum(const float* v, const float* r, int n, double* out) {
    double s = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += (double(v[i]) - r[i]) * (double(v[i]) - r[i]);
    s = warp_sum_d(s);
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int i = 0; i < (blockDim.x >> 5); ++i) t += sh[i];
        out[0] = t;
    }
}

__global__ void sum_floats(const float* x, int n, double* out) {
    double s = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
    s = warp_sum_d(s);
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0;
        for (int i = 0; i < (blockDim.x >> 5); ++i) t += sh[i];  // fixed order
        *out = t;
    }
}
__global__ void add_into(float* __restrict__ dst, const float* __restrict__ src, int64_t n) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) dst[i] += src[i];
}

#define OPPO_NCCL_CHECK(x)                                                                  \
    do {                                                                                    \
        const ncclResult_t r_ = (x);                                                        \
        if (r_ != ncclSuccess)                                                              \
            throw ::oppo::Error(OPPO_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)

// Sum-allreduce of a device buffer across the data-parallel ranks: NCCL when
// the engine has a communicator, else the host-provided callback.
void dp_allreduce(Engine& e, void* buf, int64_t count, bool f64, cudaStream_t st) {
    if (e.nccl) {
        OPPO_NCCL_CHECK(ncclAllReduce(buf, buf, static_cast<size_t>(count), f64 ? ncclDouble : ncclFloat,
                                      ncclSum, static_cast<ncclComm_t>(e.nccl), st));
        return;
    }
    if (!e.cfg.allreduce) internal_error("data-parallel update without a communicator");
    if (e.cfg.allreduce(e.cfg.allreduce_ctx, buf, count, f64 ? 1 : 0, st) != 0)
        throw Error(OPPO_ERR_NCCL, "host allreduce callback failed");
}

template <class T>
void ppo_update_impl(Engine& e, const std::vector<int>& slots, const oppo_ppo_hparams& hp,
                     oppo_ppo_stats& st_out) {
    cudaStream_t st = e.su;  // the update runs between steps: whole GPU
    ActorSms actor_sms(e);
    cudaEvent_t t0, t1;
    OPPO_CUDA_CHECK(cudaEventCreate(&t0));
    OPPO_CUDA_CHECK(cudaEventCreate(&t1));
    OPPO_CUDA_CHECK(cudaEventRecord(t0, st));
    const int n = static_cast<int>(slots.size());
    std::vector<int32_t> off(n + 1, 0), sl(slots.begin(), slots.end());
    for (int i = 0; i < n; ++i) off[i + 1] = off[i] + e.slots[slots[i]].target_len;
    const int N = off[n];
    Model& actor = e.models[ACTOR];
    Model& critic = e.models[CRITIC];
    const int Da = actor.dims.d_model, Dc = critic.dims.d_model, V = actor.dims.vocab;
    const int Npad = (N + 7) / 8 * 8;
    // device buffers (grown on demand)
    size_t meta_bytes = 0;
    for (int i = 0; i < n; ++i) meta_bytes += 16 * cdiv(e.slots[slots[i]].prompt_len + off[i + 1] - off[i], 32);
    const size_t need = static_cast<size_t>(Npad) * (4 * 14) + static_cast<size_t>(n + 1) * 20 * 4 +
                        static_cast<size_t>(Npad) * (Da + Dc) * sizeof(T) + 4096 * 8 + 1024 +
                        meta_bytes + static_cast<size_t>(n) * 16 + 16384 +
                        static_cast<size_t>(Npad + n * (e.Pmax + 1)) * 12;
    if (need > e.ppo_buf_bytes) {
        if (e.ppo_buf) cudaFree(e.ppo_buf);
        e.ppo_buf_bytes = need * 3 / 2;
        e.ppo_buf = dalloc(e.ppo_buf_bytes);
    }
    uint8_t* p = static_cast<uint8_t*>(e.ppo_buf);
    auto take = [&](size_t bytes) {
        uint8_t* r = p;
        p += (bytes + 255) & ~size_t(255);
        return r;
    };
    int32_t* d_slots = reinterpret_cast<int32_t*>(take(n * 4));
    int32_t* d_off = reinterpret_cast<int32_t*>(take((n + 1) * 4));
    int32_t* d_tokv = reinterpret_cast<int32_t*>(take(Npad * 4));
    float* d_old = reinterpret_cast<float*>(take(Npad * 4));
    float* d_ref = reinterpret_cast<float*>(take(Npad * 4));
    float* d_vtok = reinterpret_cast<float*>(take(Npad * 4));
    float* d_vals = reinterpret_cast<float*>(take((N + n) * 4));
    float* d_score = reinterpret_cast<float*>(take(n * 4));
    float* d_rew = reinterpret_cast<float*>(take(Npad * 4));
    float* d_kl = reinterpret_cast<float*>(take(Npad * 4));
    float* d_adv = reinterpret_cast<float*>(take(Npad * 4));
    float* d_ret = reinterpret_cast<float*>(take(Npad * 4));
    float* d_new = reinterpret_cast<float*>(take(Npad * 4));
    float* d_lse = reinterpret_cast<float*>(take(Npad * 4));
    float* d_dobj = reinterpret_cast<float*>(take(Npad * 4));
    double* d_part = reinterpret_cast<double*>(take(4096 * 8));
    double* d_stats = reinterpret_cast<double*>(take(16 * 8));
    T* d_hf = reinterpret_cast<T*>(take(static_cast<size_t>(Npad) * Da * sizeof(T)));
    T* d_hc = reinterpret_cast<T*>(take(static_cast<size_t>(Npad) * Dc * sizeof(T)));
    OPPO_CUDA_CHECK(cudaMemcpyAsync(d_slots, sl.data(), n * 4, cudaMemcpyHostToDevice, st));
    OPPO_CUDA_CHECK(cudaMemcpyAsync(d_off, off.data(), (n + 1) * 4, cudaMemcpyHostToDevice, st));
    OPPO_CUDA_CHECK(cudaMemsetAsync(d_tokv, 0, Npad * 4, st));
    OPPO_CUDA_CHECK(cudaMemsetAsync(d_hf, 0, static_cast<size_t>(Npad) * Da * sizeof(T), st));
    gather_batch<T><<<n, 128, 0, st>>>(d_slots, d_off, n, e.d_tok, e.d_old_lp, e.d_ref_lp, e.d_values,
                                       e.d_reward, e.tok_stride, d_tokv, d_old, d_ref, d_vtok, d_vals,
                                       d_score);
    gather_hidden<T><<<dim3(64, n), 128, 0, st>>>(d_slots, d_off, n, static_cast<const T*>(e.d_hf_actor),
                                                  e.tok_stride, Da, d_hf);
    gather_hidden<T><<<dim3(64, n), 128, 0, st>>>(d_slots, d_off, n, static_cast<const T*>(e.d_hf_critic),
                                                  e.tok_stride, Dc, d_hc);
    // K7 KL-shaped reward, K8 GAE
    token_rewards<float><<<n, 128, 0, st>>>(n, d_off, d_score, d_old, d_ref,
                                            static_cast<float>(hp.kl_coef), d_rew, d_kl);
    gae_scan<float><<<cdiv(n * 32, 128), 128, 0, st>>>(n, d_off, d_rew, d_vals,
                                                      static_cast<float>(hp.gamma),
                                                      static_cast<float>(hp.lambda), d_adv, d_ret);
    if (hp.value_target == OPPO_VALUE_MC_RETURN)  // the reference's value target (ppo.cpp:296-314)
        mc_returns<float><<<cdiv(n, 128), 128, 0, st>>>(n, d_off, d_score, static_cast<float>(hp.gamma), d_ret);
    else if (hp.value_target != OPPO_VALUE_GAE_RETURN)
        config_error("value_target must be OPPO_VALUE_MC_RETURN or OPPO_VALUE_GAE_RETURN");
    // K9 whitening statistics.  Data-parallel runs allreduce
    // {sum adv, sum adv^2, n_tokens, sum reward, n_samples} in one fp64 NCCL
    // call: whitening uses the global moments, the token mean of the
    // objective / gradients the global token count, and every rank's Delta
    // controller the global mean reward.
    // data-parallel collectives: world > 1, or a communicator given explicitly
    // (world 1 with NCCL runs every collective on one GPU: the hardware check
    // of the NCCL call sites, tests/test_gpu_dp.py)
    const bool dp = (e.cfg.world > 1 && e.cfg.allreduce != nullptr) || e.nccl != nullptr;
    const int mb = std::min(1024, std::max(1, cdiv(N, 256)));
    double* stats = nullptr;
    double n_glob = N, score_glob = 0, samples_glob = n;
    if (hp.whiten || dp) {
        moments<float><<<mb, 256, 0, st>>>(d_adv, N, d_part);
        moments_final<<<1, 32, 0, st>>>(d_part, mb, static_cast<double>(N), d_stats);
        if (hp.whiten) stats = d_stats;
    }
    if (dp) {
        sum_floats<<<1, 256, 0, st>>>(d_score, n, d_stats + 3);
        const double nn = n;
        OPPO_CUDA_CHECK(cudaMemcpyAsync(d_stats + 6, &nn, 8, cudaMemcpyHostToDevice, st));
        OPPO_CUDA_CHECK(cudaMemcpyAsync(d_stats + 4, d_stats + 6, 8, cudaMemcpyDeviceToDevice, st));
        dp_allreduce(e, d_stats, 5, true, st);
        double g[5];
        OPPO_CUDA_CHECK(cudaMemcpyAsync(g, d_stats, 5 * 8, cudaMemcpyDeviceToHost, st));
        OPPO_CUDA_CHECK(cudaStreamSynchronize(st));
        n_glob = g[2];
        score_glob = g[3];
        samples_glob = g[4];
    }
    const float inv_n_glob = 1.0f / static_cast<float>(std::max(1.0, n_glob));
    // full-parameter update (K11 / K12, train.cu): the actor's objective and the
    // critic's value loss come from the training forward of every layer
    const bool full = e.cfg.train_heads == 2;
    const bool full_actor = full && hp.learning_rate != 0, full_critic = full && hp.value_learning_rate != 0;
    // current-policy log-probs of the sampled tokens from the cached actor
    // hidden states: computed at the end of run_step while the scorers
    // finished (precompute_policy_lp) when every sequence of the batch is
    // there and the lm_head is unchanged, else here
    const int nt = gemm_logit_tiles(e.dtype, V);
    Work& w = e.ws;
    bool use_pre = !full_actor && e.pre_lp && e.pre_version == e.lm_version && n > 0;
    std::vector<int32_t> pre_src(n);
    for (int i = 0; i < n && use_pre; ++i) {
        const auto it = e.pre_index.find(e.slots[slots[i]].id);
        if (it == e.pre_index.end() || it->second.second != off[i + 1] - off[i]) use_pre = false;
        else pre_src[i] = it->second.first;
    }
    if (use_pre) {
        int32_t* d_src = reinterpret_cast<int32_t*>(take(n * 4));
        OPPO_CUDA_CHECK(cudaMemcpyAsync(d_src, pre_src.data(), n * 4, cudaMemcpyHostToDevice, st));
        OPPO_CUDA_CHECK(cudaStreamWaitEvent(st, e.ev_pre, 0));
        gather_pre_lp<<<n, 128, 0, st>>>(d_src, d_off, n, e.pre_new, e.pre_lse, d_new, d_lse);
    }
    const int chunk_rows = std::max(32, std::min(w.max_rows, static_cast<int>((static_cast<size_t>(64) << 20) / (nt * 16))));
    for (int c0 = 0; c0 < N && !use_pre && !full_actor; c0 += chunk_rows) {
        const int cn = std::min(chunk_rows, N - c0);
        EpiParams ep{};
        ep.mode = EPI_LOGITS;
        ep.partials = w.partials;
        ep.tgt_logit = w.tgt_logit;
        ep.targets = d_tokv + c0;
        gemm_run(e, w, st, d_hf + static_cast<size_t>(c0) * Da, cn, Da, Da, actor.lm_head, V, Da, ep);
        // contiguous rows: new_lp[c0 + r] = logit[target] - lse
        logits_combine<<<cdiv(cn, 4), 128, 0, st>>>(w.partials, nt, V, cn, nullptr, w.tgt_logit, nullptr,
                                                    nullptr, nullptr, d_new + c0, 0, d_lse + c0, nullptr);
    }
    // K10 clipped objective and d obj / d logp
    const int cb = std::min(1024, cdiv(N, 256));
    if (!full_actor) {
        ppo_clip<float><<<cb, 256, 0, st>>>(N, d_new, d_old, d_adv, static_cast<float>(hp.clip_epsilon),
                                            stats, 1e-8, d_dobj, d_part, inv_n_glob);
        sum_partials<<<1, 32, 0, st>>>(d_part, cb, d_stats + 4);
    } else {
        OPPO_CUDA_CHECK(cudaMemsetAsync(d_stats + 4, 0, 8, st));
    }
    float* d_sq = reinterpret_cast<float*>(take(Npad * 4));
    if (full_actor || full_critic) {
        TrainBatch tb;
        for (int i = 0; i < n; ++i) {
            tb.slot.push_back(slots[i]);
            tb.P.push_back(e.slots[slots[i]].prompt_len);
            tb.L.push_back(off[i + 1] - off[i]);
        }
        tb.off = off;
        // micro-batch rows: as many as ~36 GB of saved activations allow, in
        // steps of 4096, at most 32768 (0.5B: 32768, measured update 866 -> 838 ms
        // vs 16384 at 39K tokens; 1.5B: 16384; 7B: 4096)
        int auto_rows = 32768;
        for (int mid : {ACTOR, CRITIC}) {
            const auto& md = e.models[mid].dims;
            const double per_row = static_cast<double>(md.n_layers) *
                (2.0 * md.d_model * 4 + 2.0 * md.d_model * e.esz +
                 (static_cast<double>(md.n_heads + 2 * md.n_kv_heads) * md.head_dim + md.n_heads * md.head_dim +
                  3.0 * md.d_ff) * e.esz);
            auto_rows = std::min(auto_rows, std::max(4096, static_cast<int>((36.0 * (1 << 30)) / per_row) / 4096 * 4096));
        }
        tb.rows_max = std::max(256, env_int("OPPO_TRAIN_ROWS", auto_rows));
        tb.tok = d_tokv;
        tb.adv = d_adv;
        tb.old_lp = d_old;
        tb.ret = d_ret;
        tb.new_lp = d_new;
        tb.lse = d_lse;
        tb.dobj = d_dobj;
        tb.stats = stats;
        tb.clip_eps = static_cast<float>(hp.clip_epsilon);
        tb.inv_n = inv_n_glob;
        tb.part = d_part;
        tb.obj_acc = d_stats + 4;
        tb.sq = d_sq;
        // micro-batch metadata: sequences, 32-row attention blocks, response-row map
        size_t blocks = 0;
        for (int i = 0; i < n; ++i) blocks += cdiv(tb.P[i] + tb.L[i] - 1, 32);
        size_t rows_all = 0;
        for (int i = 0; i < n; ++i) rows_all += tb.P[i] + tb.L[i] - 1;
        tb.meta_cap = static_cast<size_t>(n) * 16 + blocks * 16 + static_cast<size_t>(N) * 4 + rows_all * 12 + 8192;
        tb.meta_dev = take(tb.meta_cap);
        if (e.dtype == OPPO_DTYPE_F32) train_full<float>(e, tb, hp, dp, st);
        else train_full<__nv_bfloat16>(e, tb, hp, dp, st);
        if (full_actor) ++e.lm_version;
    }
    // K11 head update: lm_head += lr * dObj/dW  (gradient ascent, ppo.cpp:288-290)
    if (e.cfg.train_heads == 1 && hp.learning_rate > 0) {
        const int gc = e.g_chunk;
        if (!e.g_buf) {
            e.g_buf = dalloc(static_cast<size_t>(V) * gc * sizeof(T));
            e.ht_buf = dalloc(static_cast<size_t>(std::max(Da, Dc)) * gc * sizeof(T));
            e.vgrad = static_cast<float*>(dalloc(std::max(Da, Dc) * 4));
        }
        // DP: accumulate lr * dObj/dW into a gradient buffer, allreduce it, then
        // apply; single GPU: accumulate straight into the fp32 master
        const size_t nw = static_cast<size_t>(V) * Da;
        float* gdst = actor.lm_master;
        if (dp) {
            if (!e.g_lm) e.g_lm = static_cast<float*>(dalloc(nw * 4));
            OPPO_CUDA_CHECK(cudaMemsetAsync(e.g_lm, 0, nw * 4, st));
            gdst = e.g_lm;
        }
        for (int c0 = 0; c0 < N; c0 += gc) {
            const int cn = std::min(gc, N - c0);
            const int cp = (cn + 7) / 8 * 8;
            EpiParams ep{};
            ep.mode = EPI_SOFTMAX_GRAD;
            ep.y = e.g_buf;
            ep.ldy = cp;
            ep.lse = d_lse + c0;
            ep.coef = d_dobj + c0;
            ep.targets = d_tokv + c0;
            if (cp != cn) OPPO_CUDA_CHECK(cudaMemsetAsync(e.g_buf, 0, static_cast<size_t>(V) * cp * sizeof(T), st));
            gemm_run(e, w, st, d_hf + static_cast<size_t>(c0) * Da, cn, Da, Da, actor.lm_head, V, Da, ep);
            transpose_rows<T><<<dim3(cdiv(Da, 32), cdiv(cp, 32)), dim3(32, 8), 0, st>>>(
                d_hf + static_cast<size_t>(c0) * Da, cn, Da, cp, static_cast<T*>(e.ht_buf));
            EpiParams eg{};
            eg.mode = EPI_ADD_F32;
            eg.y = gdst;
            eg.ldy = Da;
            eg.scale = static_cast<float>(hp.learning_rate);
            gemm_run(e, w, st, e.g_buf, V, cp, cp, e.ht_buf, Da, cp, eg);
        }
        if (dp) {  // gradient allreduce (sum: every rank's dObj already carries 1/N_global)
            dp_allreduce(e, e.g_lm, static_cast<int64_t>(nw), false, st);
            add_into<<<cdiv(static_cast<int64_t>(nw), 256), 256, 0, st>>>(actor.lm_master, e.g_lm,
                                                                        static_cast<int64_t>(nw));
        }
        const size_t nn = nw;
        convert<float, T><<<cdiv(nn, 256), 256, 0, st>>>(actor.lm_master, static_cast<T*>(actor.lm_head), nn);
        ++e.lm_version;  // precomputed policy log-probs are stale from here
        // critic value head: w -= vlr * (1/N) sum (V - R) h
        value_head_grad<T><<<cdiv(Dc, 128), 128, 0, st>>>(d_hc, Dc, N, d_vtok, d_ret, e.vgrad, inv_n_glob);
        if (dp)
            dp_allreduce(e, e.vgrad, Dc, false, st);
        head_sgd<<<cdiv(Dc, 128), 128, 0, st>>>(critic.head, e.vgrad, Dc,
                                                static_cast<float>(hp.value_learning_rate));
    }
    if (full_critic) {  // value loss of the critic's training forward
        OPPO_CUDA_CHECK(cudaMemsetAsync(d_stats + 5, 0, 8, st));
        train::sum_to_double<<<1, 256, 0, st>>>(d_sq, N, d_stats + 5);
    } else {
        sq_err_sum<<<1, 256, 0, st>>>(d_vtok, d_ret, N, d_stats + 5);
    }
    // statistics back to the host
    double hs[8] = {0};
    OPPO_CUDA_CHECK(cudaMemcpyAsync(hs, d_stats, 8 * 8, cudaMemcpyDeviceToHost, st));
    std::vector<float> score(n), kl(N);
    OPPO_CUDA_CHECK(cudaMemcpyAsync(score.data(), d_score, n * 4, cudaMemcpyDeviceToHost, st));
    OPPO_CUDA_CHECK(cudaMemcpyAsync(kl.data(), d_kl, N * 4, cudaMemcpyDeviceToHost, st));
    OPPO_CUDA_CHECK(cudaEventRecord(t1, st));
    OPPO_CUDA_CHECK(cudaEventSynchronize(t1));
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    st_out = {};
    double sr = 0, sk = 0;
    for (float x : score) sr += x;
    for (float x : kl) sk += x;
    st_out.mean_reward = n ? sr / n : 0.0;
    if (dp) st_out.mean_reward = samples_glob > 0 ? score_glob / samples_glob : 0.0;  // global mean
    st_out.kl_mean = N ? sk / N : 0.0;
    st_out.ppo_objective = N ? hs[4] / N : 0.0;
    st_out.value_loss = N ? 0.5 * hs[5] / N : 0.0;
    if (hp.whiten && N) {
        st_out.adv_mean = hs[0] / N;
        st_out.adv_std = std::sqrt(std::max(0.0, hs[1] / N - st_out.adv_mean * st_out.adv_mean));
    }
    st_out.n_tokens = N;
    st_out.n_samples = n;
    st_out.update_us = ms * 1e3;
}

}  // namespace

void dp_allreduce_pub(Engine& e, void* buf, int64_t count, bool f64, cudaStream_t st) {
    dp_allreduce(e, buf, count, f64, st);
}

// One gradient bucket (fp32 tensors): a single NCCL group launch when the
// engine has a communicator (the tensors of a layer travel as one fused
// collective), else one host-callback allreduce per tensor.
void dp_allreduce_bucket(Engine& e, const std::vector<std::pair<float*, int64_t>>& bufs, cudaStream_t st) {
    if (e.nccl) {
        OPPO_NCCL_CHECK(ncclGroupStart());
        for (const auto& b : bufs)
            OPPO_NCCL_CHECK(ncclAllReduce(b.first, b.first, static_cast<size_t>(b.second), ncclFloat, ncclSum,
                                          static_cast<ncclComm_t>(e.nccl), st));
        OPPO_NCCL_CHECK(ncclGroupEnd());
        return;
    }
    for (const auto& b : bufs) dp_allreduce(e, b.first, b.second, false, st);
}

}  // namespace oppo

// ==================================================================== C ABI
namespace oppo {
namespace {

template <class F>
oppo_status eguard(Engine* e, F&& f) {
    try {
        f();
        return OPPO_OK;
    } catch (const Error& x) {
        if (e) e->error = x.what();
        return x.code;
    } catch (const std::exception& x) {
        if (e) e->error = x.what();
        return OPPO_ERR_INTERNAL;
    }
}

// ----------------------------------------------------------- checkpoints
// Engine state between steps (the carry buffer's device side +
// KV page tables): which slots hold which sequences, their pages, prompts,
// tokens / log-probs / values / rewards / cached hidden states, the KV pages
// they own in every model's pool, and the trained heads.  Weights that are
// not trained are regenerated from the engine's weight seed, so a checkpoint
// loads into a fresh engine created with the same configuration.
constexpr char kCkptMagic[8] = {'O', 'P', 'P', 'O', 'C', 'K', 'P', '1'};

struct CkptSig {  // configuration fields a checkpoint depends on
    oppo_model_dims dims[N_MODELS];
    int32_t dtype, S, Pmax, Lmax, page_size, n_pages, train_heads, carry;
    uint64_t weight_seed, sample_seed;
};

CkptSig ckpt_sig(const Engine& e) {
    CkptSig g;
    std::memset(&g, 0, sizeof(g));
    for (int i = 0; i < N_MODELS; ++i) g.dims[i] = e.models[i].dims;
    g.dtype = e.dtype;
    g.S = e.S;
    g.Pmax = e.Pmax;
    g.Lmax = e.Lmax;
    g.page_size = e.page_size;
    g.n_pages = e.n_pages;
    g.train_heads = e.cfg.train_heads;
    g.carry = e.cfg.carry_granularity;
    g.weight_seed = e.cfg.weight_seed;
    g.sample_seed = e.cfg.sample_seed;
    return g;
}

struct CkptFile {
    std::FILE* f;
    bool writing;
    CkptFile(const char* path, bool w) : f(std::fopen(path, w ? "wb" : "rb")), writing(w) {
        if (!f) input_error(std::string("cannot open checkpoint ") + path);
    }
    ~CkptFile() {
        if (f) std::fclose(f);
    }
    void raw(void* p, size_t n) {
        const size_t k = writing ? std::fwrite(p, 1, n, f) : std::fread(p, 1, n, f);
        if (k != n) input_error(writing ? "checkpoint write failed" : "checkpoint truncated");
    }
    template <class V>
    void pod(V& v) {
        raw(&v, sizeof(V));
    }
    template <class V>
    void vec(std::vector<V>& v) {
        uint64_t n = v.size();
        pod(n);
        if (!writing) {
            if (n > (uint64_t(1) << 32)) input_error("checkpoint corrupt");
            v.resize(n);
        }
        if (n) raw(v.data(), n * sizeof(V));
    }
    // device range through a host staging buffer
    void dev(void* d, size_t n) {
        std::vector<uint8_t> h(n);
        if (writing) OPPO_CUDA_CHECK(cudaMemcpy(h.data(), d, n, cudaMemcpyDeviceToHost));
        raw(h.data(), n);
        if (!writing) OPPO_CUDA_CHECK(cudaMemcpy(d, h.data(), n, cudaMemcpyHostToDevice));
    }
    // rows [0, layers) of `width` bytes, `pitch` bytes apart (one KV page over all layers)
    void dev2d(void* d, size_t pitch, size_t width, size_t rows) {
        std::vector<uint8_t> h(width * rows);
        if (writing) OPPO_CUDA_CHECK(cudaMemcpy2D(h.data(), width, d, pitch, width, rows, cudaMemcpyDeviceToHost));
        raw(h.data(), h.size());
        if (!writing) OPPO_CUDA_CHECK(cudaMemcpy2D(d, pitch, h.data(), width, width, rows, cudaMemcpyHostToDevice));
    }
};

// One routine for both directions keeps the file layout in one place.
void checkpoint_io(Engine& e, CkptFile& io) {
    if (e.step_open) input_error("checkpoint inside an open step");
    OPPO_CUDA_CHECK(cudaDeviceSynchronize());
    char magic[8];
    std::memcpy(magic, kCkptMagic, 8);
    io.raw(magic, 8);
    if (std::memcmp(magic, kCkptMagic, 8) != 0) input_error("not an oppo checkpoint");
    CkptSig sig = ckpt_sig(e), cur = sig;
    io.pod(sig);
    if (std::memcmp(&sig, &cur, sizeof(sig)) != 0)
        config_error("checkpoint was written by an engine with another configuration");
    if (!io.writing && !e.slot_of.empty()) input_error("checkpoint load needs an engine without sequences");
    // host state
    io.pod(e.lm_version);
    io.vec(e.free_slots);
    io.vec(e.free_pages);
    std::vector<int32_t> live;
    if (io.writing)
        for (int s = 0; s < e.S; ++s)
            if (e.slots[s].id >= 0) live.push_back(s);
    io.vec(live);
    for (int s : live) {
        if (s < 0 || s >= e.S) input_error("checkpoint corrupt");
        auto& info = e.slots[s];
        int32_t flags = (info.ref_pending ? 1 : 0) | (info.scored_prompt ? 2 : 0);
        io.pod(info.id);
        io.pod(info.prompt_len);
        io.pod(info.target_len);
        io.pod(flags);
        io.vec(info.pages);
        if (!io.writing) {
            info.ref_pending = flags & 1;
            info.scored_prompt = flags & 2;
            e.slot_of[info.id] = s;
        }
    }
    // per-slot device arrays (whole: a few MB), cached hidden rows of live slots
    const size_t S1 = e.S + 1, TS = e.tok_stride;
    io.dev(e.d_page_table, S1 * e.max_pages * 4);
    io.dev(e.d_prompt, S1 * e.Pmax * 4);
    io.dev(e.d_tok, S1 * TS * 4);
    io.dev(e.d_old_lp, S1 * TS * 4);
    io.dev(e.d_ref_lp, S1 * TS * 4);
    io.dev(e.d_values, S1 * TS * 4);
    io.dev(e.d_reward, S1 * 4);
    io.dev(e.d_target_len, S1 * 4);
    io.dev(e.d_ref_pending, S1 * e.models[REF].dims.d_model * e.esz);
    for (int s : live) {
        const size_t ra = TS * e.models[ACTOR].dims.d_model * e.esz, rc = TS * e.models[CRITIC].dims.d_model * e.esz;
        io.dev(static_cast<uint8_t*>(e.d_hf_actor) + s * ra, ra);
        io.dev(static_cast<uint8_t*>(e.d_hf_critic) + s * rc, rc);
    }
    // KV pages owned by live slots, every model and layer
    for (auto& m : e.models) {
        if (!m.used) continue;
        const size_t page_elems = static_cast<size_t>(m.dims.n_kv_heads) * e.page_size * m.dims.head_dim;
        for (int s : live)
            for (int pg : e.slots[s].pages)
                for (void* pool : {m.k_pool, m.v_pool})
                    io.dev2d(static_cast<uint8_t*>(pool) + pg * page_elems * e.esz, m.layer_stride * e.esz,
                             page_elems * e.esz, m.dims.n_layers);
    }
    // trained tensors: every actor / critic tensor and its fp32 master (full
    // update), or the heads
    if (e.cfg.train_heads == 2) {
        for (auto& [ptr, bytes] : train_tensors(e, e.su)) io.dev(ptr, bytes);
    } else if (e.cfg.train_heads) {
        Model& a = e.models[ACTOR];
        const size_t nw = static_cast<size_t>(a.dims.vocab) * a.dims.d_model;
        io.dev(a.lm_head, nw * e.esz);
        if (a.lm_master) io.dev(a.lm_master, nw * 4);
        io.dev(e.models[CRITIC].head, e.models[CRITIC].dims.d_model * 4);
    }
    if (!io.writing) {
        e.pre_version = -1;  // precomputed policy log-probs are not part of a checkpoint
        e.pre_index.clear();
    }
}

void release_slot(Engine& e, int64_t id) {
    auto it = e.slot_of.find(id);
    if (it == e.slot_of.end()) input_error("release of unknown sequence " + std::to_string(id));
    auto& info = e.slots[it->second];
    for (int p : info.pages) e.free_pages.push_back(p);
    info = SlotInfo{};
    e.free_slots.push_back(it->second);
    e.slot_of.erase(it);
}

struct EngineHooks final : LoopHooks {
    Engine& e;
    oppo_ppo_hparams hp;
    oppo_prompt_fn prompt = nullptr;
    void* prompt_ctx = nullptr;
    int reserved_slots = 0, reserved_pages = 0;
    explicit EngineHooks(Engine& en, const oppo_ppo_hparams& h) : e(en), hp(h) {}
    void admit(const std::vector<oppo_seq_state>& fresh) override {
        if (fresh.empty()) return;
        std::vector<int32_t> tok;
        if (prompt) {  // the caller's prompt source (PromptSource::next, overcommit.hpp:16-20)
            for (const auto& s : fresh) {
                const size_t o = tok.size();
                tok.resize(o + s.prompt_len);
                if (prompt(prompt_ctx, s.id, s.prompt_len, tok.data() + o) != 0)
                    input_error("prompt source failed for sequence " + std::to_string(s.id));
            }
        }
        const int32_t* p = prompt ? tok.data() : nullptr;
        if (e.dtype == OPPO_DTYPE_F32) admit_impl<float>(e, fresh.data(), static_cast<int>(fresh.size()), p);
        else admit_impl<__nv_bfloat16>(e, fresh.data(), static_cast<int>(fresh.size()), p);
    }
    int rank() const override { return e.cfg.world > 1 ? e.cfg.rank : 0; }
    int world() const override { return std::max(1, e.cfg.world); }
    bool dp() const { return e.cfg.world > 1 && (e.nccl != nullptr || e.cfg.allreduce != nullptr); }
    // oppo_ppo_update allreduces the reward statistics itself when data parallel
    bool reward_is_global() const override { return e.cfg.world <= 1 || dp(); }
    void allreduce_sum(double* v, int n) override {
        if (e.cfg.world <= 1) return;
        if (!dp()) config_error("world > 1 without a communicator (nccl_comm or allreduce hook)");
        double* d = nullptr;
        OPPO_CUDA_CHECK(cudaMalloc(&d, n * sizeof(double)));
        OPPO_CUDA_CHECK(cudaMemcpyAsync(d, v, n * sizeof(double), cudaMemcpyHostToDevice, e.su));
        dp_allreduce(e, d, n, true, e.su);
        OPPO_CUDA_CHECK(cudaMemcpyAsync(v, d, n * sizeof(double), cudaMemcpyDeviceToHost, e.su));
        OPPO_CUDA_CHECK(cudaStreamSynchronize(e.su));
        cudaFree(d);
    }
    // KV admission control: a sequence is admitted only with a free slot and
    // KV pages for prompt + target length (else refill defers it)
    void begin_refill() override { reserved_slots = reserved_pages = 0; }
    bool fits(const oppo_seq_state& s) override {
        const int need = cdiv(s.prompt_len + s.target_len + 1, e.page_size);
        if (reserved_slots + 1 > static_cast<int>(e.free_slots.size()) ||
            reserved_pages + need > static_cast<int>(e.free_pages.size()))
            return false;
        ++reserved_slots;
        reserved_pages += need;
        return true;
    }
    void execute(const std::vector<oppo_seq_state>& active, int chunk, int mode, int stop,
                 std::vector<oppo_seq_outcome>& out, oppo_ledger& ledger) override {
        if (e.dtype == OPPO_DTYPE_F32) run_step_impl<float>(e, active, chunk, mode, stop, out, ledger);
        else run_step_impl<__nv_bfloat16>(e, active, chunk, mode, stop, out, ledger);
    }
    double update(const std::vector<oppo_seq_state>& batch, bool train, oppo_step_record& rec) override {
        if (!train || batch.empty()) return 0.0;
        std::vector<int> slots;
        for (const auto& s : batch) slots.push_back(e.slot_of.at(s.id));
        oppo_ppo_stats st{};
        if (e.dtype == OPPO_DTYPE_F32) ppo_update_impl<float>(e, slots, hp, st);
        else ppo_update_impl<__nv_bfloat16>(e, slots, hp, st);
        rec.update_us = st.update_us;
        rec.ppo_loss = st.ppo_objective;
        rec.kl_mean = st.kl_mean;
        rec.batch_tokens = st.n_tokens;
        return st.mean_reward;
    }
    void release(const std::vector<oppo_seq_state>& batch) override {
        for (const auto& s : batch) release_slot(e, s.id);
    }
};

}  // namespace
}  // namespace oppo

using oppo::Engine;

extern "C" {

oppo_status oppo_engine_create(const oppo_engine_cfg* cfg, oppo_engine** out) {
    *out = nullptr;
    try {
        *out = reinterpret_cast<oppo_engine*>(oppo::engine_new(*cfg));
        return OPPO_OK;
    } catch (const oppo::Error& x) {
        oppo_set_global_error(x.what());
        return x.code;
    } catch (const std::exception& x) {
        oppo_set_global_error(x.what());
        return OPPO_ERR_INTERNAL;
    }
}

void oppo_engine_destroy(oppo_engine* e) { oppo::engine_free(reinterpret_cast<Engine*>(e)); }

const char* oppo_last_error(const oppo_engine* e) {
    return e ? reinterpret_cast<const Engine*>(e)->error.c_str() : oppo_last_error_global();
}

oppo_status oppo_admit(oppo_engine* eh, const oppo_seq_state* seqs, int32_t n,
                       const int32_t* prompt_tokens) {
    Engine* e = reinterpret_cast<Engine*>(eh);
    return oppo::eguard(e, [&] {
        if (e->dtype == OPPO_DTYPE_F32) oppo::admit_impl<float>(*e, seqs, n, prompt_tokens);
        else oppo::admit_impl<__nv_bfloat16>(*e, seqs, n, prompt_tokens);
    });
}

oppo_status oppo_run_step(oppo_engine* eh, const oppo_seq_state* active, int32_t n_active,
                          int32_t chunk_size, int32_t mode, int32_t stop_after,
                          oppo_seq_outcome* out, oppo_ledger* ledger) {
    Engine* e = reinterpret_cast<Engine*>(eh);
    return oppo::eguard(e, [&] {
        std::vector<oppo_seq_state> v(active, active + n_active);
        std::vector<oppo_seq_outcome> o;
        oppo_ledger l{};
        if (e->dtype == OPPO_DTYPE_F32) oppo::run_step_impl<float>(*e, v, chunk_size, mode, stop_after, o, l);
        else oppo::run_step_impl<__nv_bfloat16>(*e, v, chunk_size, mode, stop_after, o, l);
        std::copy(o.begin(), o.end(), out);
        *ledger = l;
    });
}

oppo_status oppo_ppo_update(oppo_engine* eh, const int64_t* ids, int32_t n,
                            const oppo_ppo_hparams* hp, oppo_ppo_stats* out) {
    Engine* e = reinterpret_cast<Engine*>(eh);
    return oppo::eguard(e, [&] {
        std::vector<int> slots;
        for (int i = 0; i < n; ++i) {
            auto it = e->slot_of.find(ids[i]);
            if (it == e->slot_of.end()) oppo::input_error("update of unknown sequence");
            slots.push_back(it->second);
        }
        if (e->dtype == OPPO_DTYPE_F32) oppo::ppo_update_impl<float>(*e, slots, *hp, *out);
        else oppo::ppo_update_impl<__nv_bfloat16>(*e, slots, *hp, *out);
    });
}

oppo_status oppo_engine_save(oppo_engine* eh, const char* path) {
    Engine* e = reinterpret_cast<Engine*>(eh);
    return oppo::eguard(e, [&] {
        oppo::CkptFile io(path, true);
        oppo::checkpoint_io(*e, io);
    });
}

oppo_status oppo_engine_load(oppo_engine* eh, const char* path) {
    Engine* e = reinterpret_cast<Engine*>(eh);
    return oppo::eguard(e, [&] {
        oppo::CkptFile io(path, false);
        oppo::checkpoint_io(*e, io);
    });
}

oppo_status oppo_release(oppo_engine* eh, const int64_t* ids, int32_t n) {
    Engine* e = reinterpret_cast<Engine*>(eh);
    return oppo::eguard(e, [&] {
        for (int i = 0; i < n; ++i) oppo::release_slot(*e, ids[i]);
    });
}

oppo_status oppo_read_rollout(oppo_engine* eh, int64_t id, int32_t* tokens, float* old_lp,
                              float* ref_lp, float* values, float* reward, int32_t cap,
                              int32_t* len) {
    Engine* e = reinterpret_cast<Engine*>(eh);
    return oppo::eguard(e, [&] {
        auto it = e->slot_of.find(id);
        if (it == e->slot_of.end()) oppo::input_error("unknown sequence");
        const int s = it->second;
        const int L = e->slots[s].target_len;
        *len = L;
        if (cap < L + 2) oppo::input_error("buffer too small");
        OPPO_CUDA_CHECK(cudaStreamSynchronize(e->sa));
        OPPO_CUDA_CHECK(cudaStreamSynchronize(e->ss));
        const size_t o = static_cast<size_t>(s) * e->tok_stride;
        if (tokens) OPPO_CUDA_CHECK(cudaMemcpy(tokens, e->d_tok + o, (L + 1) * 4, cudaMemcpyDeviceToHost));
        if (old_lp) OPPO_CUDA_CHECK(cudaMemcpy(old_lp, e->d_old_lp + o, (L + 1) * 4, cudaMemcpyDeviceToHost));
        if (ref_lp) OPPO_CUDA_CHECK(cudaMemcpy(ref_lp, e->d_ref_lp + o, (L + 1) * 4, cudaMemcpyDeviceToHost));
        if (values) OPPO_CUDA_CHECK(cudaMemcpy(values, e->d_values + o, (L + 2) * 4, cudaMemcpyDeviceToHost));
        if (reward) OPPO_CUDA_CHECK(cudaMemcpy(reward, e->d_reward + s, 4, cudaMemcpyDeviceToHost));
    });
}

oppo_status oppo_read_prompt(oppo_engine* eh, int64_t id, int32_t* out, int32_t cap, int32_t* len) {
    Engine* e = reinterpret_cast<Engine*>(eh);
    return oppo::eguard(e, [&] {
        auto it = e->slot_of.find(id);
        if (it == e->slot_of.end()) oppo::input_error("unknown sequence");
        const int s = it->second, P = e->slots[s].prompt_len;
        *len = P;
        if (cap < P) oppo::input_error("buffer too small");
        OPPO_CUDA_CHECK(cudaStreamSynchronize(e->sa));
        OPPO_CUDA_CHECK(cudaMemcpy(out, e->d_prompt + static_cast<size_t>(s) * e->Pmax, P * 4,
                                   cudaMemcpyDeviceToHost));
    });
}

// Copies one weight tensor of a model to host as fp32 (oracle parity).
// name: embed lm_head final_norm head wqkv bqkv wo wgu wdown ln1 ln2
oppo_status oppo_get_tensor(oppo_engine* eh, int32_t model, const char* name, int32_t layer,
                            float* out, int64_t cap, int64_t* n_out) {
    Engine* e = reinterpret_cast<Engine*>(eh);
    return oppo::eguard(e, [&] {
        if (model < 0 || model >= oppo::N_MODELS) oppo::input_error("bad model id");
        auto& m = e->models[model];
        const auto& d = m.dims;
        std::string nm(name);
        // "<tensor>:master": the fp32 master of a bf16 matrix trained by the
        // full-parameter update (else the tensor itself)
        bool want_master = false;
        if (nm.size() > 7 && nm.compare(nm.size() - 7, 7, ":master") == 0) {
            want_master = true;
            nm.resize(nm.size() - 7);
        }
        const void* ptr = nullptr;
        int64_t n = 0;
        bool is_f32 = false;
        const int64_t D = d.d_model;
        if (nm == "embed") { ptr = m.embed; n = d.vocab * D; }
        else if (nm == "lm_head") { ptr = m.lm_head; n = d.vocab * D; }
        else if (nm == "final_norm") { ptr = m.final_norm; n = D; is_f32 = true; }
        else if (nm == "head") { ptr = m.head; n = m.head ? D : 0; is_f32 = true; }
        else {
            if (layer < 0 || layer >= d.n_layers) oppo::input_error("bad layer");
            const auto& L = m.layers[layer];
            if (nm == "wqkv") { ptr = L.wqkv; n = m.qkv_width() * D; }
            else if (nm == "bqkv") { ptr = L.bqkv; n = m.qkv_width(); is_f32 = true; }
            else if (nm == "wo") { ptr = L.wo; n = D * m.q_width(); }
            else if (nm == "wgu") { ptr = L.wgu; n = 2 * d.d_ff * D; }
            else if (nm == "wdown") { ptr = L.wdown; n = D * d.d_ff; }
            else if (nm == "ln1") { ptr = L.ln1; n = D; is_f32 = true; }
            else if (nm == "ln2") { ptr = L.ln2; n = D; is_f32 = true; }
            else oppo::input_error("unknown tensor " + nm);
        }
        if (want_master)
            if (const float* mp = oppo::train_master(*e, model, nm, layer)) {
                ptr = mp;
                is_f32 = true;
            }
        *n_out = n;
        if (!ptr || n == 0 || !out) return;  // size query
        if (cap < n) oppo::input_error("buffer too small");
        OPPO_CUDA_CHECK(cudaDeviceSynchronize());
        if (is_f32 || e->dtype == OPPO_DTYPE_F32) {
            OPPO_CUDA_CHECK(cudaMemcpy(out, ptr, n * 4, cudaMemcpyDeviceToHost));
        } else {
            float* tmp = nullptr;
            OPPO_CUDA_CHECK(cudaMalloc(&tmp, n * 4));
            oppo::convert<__nv_bfloat16, float><<<(n + 255) / 256, 256>>>(
                static_cast<const __nv_bfloat16*>(ptr), tmp, n);
            OPPO_CUDA_CHECK(cudaMemcpy(out, tmp, n * 4, cudaMemcpyDeviceToHost));
            cudaFree(tmp);
        }
    });
}

oppo_status oppo_run_seed(oppo_engine* eh, const oppo_run_config* cfg, uint64_t seed,
                          oppo_step_record* records, int32_t* n_records, int64_t* sel_ids) {
    return oppo_run_seed_ex(eh, cfg, seed, nullptr, records, n_records, sel_ids);
}

oppo_status oppo_run_seed_ex(oppo_engine* eh, const oppo_run_config* cfg, uint64_t seed,
                             const oppo_loop_hooks* lh, oppo_step_record* records, int32_t* n_records,
                             int64_t* sel_ids) {
    Engine* e = reinterpret_cast<Engine*>(eh);
    std::string err;
    const oppo_status st = oppo::eguard(e, [&] {
        oppo::EngineHooks hooks(*e, cfg->ppo);
        if (cfg->carry_granularity != e->cfg.carry_granularity)
            oppo::config_error("run config and engine disagree on carry_granularity");
        oppo::LoopExtras ex;
        if (lh) {
            hooks.prompt = lh->prompt;
            hooks.prompt_ctx = lh->prompt_ctx;
            ex.on_step = lh->on_step;
            ex.step_ctx = lh->step_ctx;
            ex.ledgers = lh->ledgers;
        }
        *n_records = oppo::run_seed_loop(*cfg, seed, hooks, records, sel_ids, &err, ex);
        // sequences still buffered at the end keep their slots; free them
        std::vector<int64_t> left;
        for (auto& kv : e->slot_of) left.push_back(kv.first);
        for (auto id : left) oppo::release_slot(*e, id);
    });
    if (st != OPPO_OK) return st;
    if (!err.empty()) {
        e->error = err;
        return OPPO_ERR_INTERNAL;
    }
    return OPPO_OK;
}

oppo_status oppo_k_ppo_token(int32_t is_f64, int32_t n_seq, const int32_t* d_off,
                             const void* d_score, const void* d_token_rewards, const void* d_values,
                             const void* d_new_lp, const void* d_old_lp, double gamma, double lambda,
                             double eps, int32_t whiten, void* d_adv, void* d_returns,
                             void* d_dobj, void* d_obj_sum, void* stream) {
    try {
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        std::vector<int32_t> off(n_seq + 1);
        OPPO_CUDA_CHECK(cudaMemcpy(off.data(), d_off, (n_seq + 1) * 4, cudaMemcpyDeviceToHost));
        const int N = off[n_seq];
        double* part = nullptr;
        OPPO_CUDA_CHECK(cudaMalloc(&part, 4096 * 8 + 64));
        double* stats = part + 4096;
        const int cb = std::max(1, std::min(1024, (N + 255) / 256));
        auto run = [&](auto tag) {
            using R = decltype(tag);
            R* rew = static_cast<R*>(const_cast<void*>(d_token_rewards));
            if (d_score) {  // terminal rewards from per-sequence scores (ppo.cpp:87-91)
                OPPO_CUDA_CHECK(cudaMalloc(&rew, std::max(1, N) * sizeof(R)));
                oppo::token_rewards<R><<<n_seq, 128, 0, st>>>(n_seq, d_off, static_cast<const R*>(d_score),
                                                              nullptr, nullptr, R(0), rew, nullptr);
            }
            oppo::gae_scan<R><<<(n_seq * 32 + 127) / 128, 128, 0, st>>>(
                n_seq, d_off, rew, static_cast<const R*>(d_values), static_cast<R>(gamma),
                static_cast<R>(lambda), static_cast<R*>(d_adv), static_cast<R*>(d_returns));
            const double* sp = nullptr;
            if (whiten) {
                oppo::moments<R><<<cb, 256, 0, st>>>(static_cast<R*>(d_adv), N, part);
                oppo::moments_final<<<1, 32, 0, st>>>(part, cb, double(N), stats);
                sp = stats;
            }
            if (d_new_lp) {
                oppo::ppo_clip<R><<<cb, 256, 0, st>>>(N, static_cast<const R*>(d_new_lp),
                                                      static_cast<const R*>(d_old_lp),
                                                      static_cast<R*>(d_adv), static_cast<R>(eps), sp,
                                                      1e-8, static_cast<R*>(d_dobj), part,
                                                      R(1) / static_cast<R>(std::max(1, N)));
                oppo::sum_partials<<<1, 32, 0, st>>>(part, cb, static_cast<double*>(d_obj_sum));
            }
            OPPO_CUDA_CHECK(cudaStreamSynchronize(st));
            if (d_score) cudaFree(rew);
        };
        if (is_f64) run(double{});
        else run(float{});
        cudaFree(part);
        OPPO_CUDA_CHECK(cudaGetLastError());
        return OPPO_OK;
    } catch (const oppo::Error& x) {
        oppo_set_global_error(x.what());
        return x.code;
    }
}

oppo_status oppo_k_gemm(int32_t dtype, int32_t M, int32_t N, int32_t K, const void* d_x,
                        const void* d_w, const void* d_bias, void* d_y, int32_t epilogue,
                        void* stream) {
    try {
        oppo::gemm_standalone(dtype, M, N, K, d_x, d_w, static_cast<const float*>(d_bias), d_y,
                              epilogue, static_cast<cudaStream_t>(stream));
        OPPO_CUDA_CHECK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
        return OPPO_OK;
    } catch (const oppo::Error& x) {
        oppo_set_global_error(x.what());
        return x.code;
    }
}

oppo_status oppo_k_gemm_t(int32_t dtype, int32_t M, int32_t N, int32_t K, const void* d_a, int32_t a_mn,
                          int32_t lda, const void* d_b, int32_t b_mn, int32_t ldb, void* d_y, int32_t epilogue,
                          void* stream) {
    try {
        if (epilogue != oppo::EPI_STORE && epilogue != oppo::EPI_ADD_F32 && epilogue != oppo::EPI_STORE_F32)
            oppo::input_error("oppo_k_gemm_t: epilogue must be 0 (store), 1 (add f32) or 5 (store f32)");
        oppo::gemm_standalone_t(dtype, M, N, K, d_a, a_mn, lda, d_b, b_mn, ldb, d_y, epilogue,
                                static_cast<cudaStream_t>(stream));
        OPPO_CUDA_CHECK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
        return OPPO_OK;
    } catch (const oppo::Error& x) {
        oppo_set_global_error(x.what());
        return x.code;
    }
}

oppo_status oppo_nccl_unique_id(uint8_t* out) {
    try {
        static_assert(sizeof(ncclUniqueId) == OPPO_NCCL_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId id;
        OPPO_NCCL_CHECK(ncclGetUniqueId(&id));
        std::memcpy(out, &id, sizeof(id));
        return OPPO_OK;
    } catch (const oppo::Error& x) {
        oppo_set_global_error(x.what());
        return x.code;
    }
}

oppo_status oppo_nccl_comm_create(const uint8_t* id, int32_t world, int32_t rank, int32_t device,
                                  void** comm) {
    try {
        if (world < 1 || rank < 0 || rank >= world) oppo::config_error("rank/world out of range");
        OPPO_CUDA_CHECK(cudaSetDevice(device));
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        ncclComm_t c;
        OPPO_NCCL_CHECK(ncclCommInitRank(&c, world, uid, rank));
        *comm = c;
        return OPPO_OK;
    } catch (const oppo::Error& x) {
        oppo_set_global_error(x.what());
        return x.code;
    }
}

oppo_status oppo_nccl_comm_destroy(void* comm) {
    if (comm) ncclCommDestroy(static_cast<ncclComm_t>(comm));
    return OPPO_OK;
}

// Decode GEMM (gemm_dec.cuh) alone: mode 0 partials (d_ws [splits][M][N] fp32,
// *splits receives the split count), 1 SwiGLU (d_y [M][N/2] bf16), 2 store
// (+bias, d_y [M][N] bf16).
oppo_status oppo_k_gemm_dec(int32_t M, int32_t N, int32_t K, const void* d_x, const void* d_w,
                            const void* d_bias, void* d_y, int32_t mode, void* d_ws,
                            int64_t ws_floats, int32_t* splits, void* stream) {
    try {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int ldy = mode == oppo::DEC_SWIGLU ? N / 2 : N;
        const int sp = oppo::gemm_dec_impl(nullptr, static_cast<cudaStream_t>(stream), d_x, M, K, K, d_w, N,
                                           K, mode, d_y, ldy, static_cast<const float*>(d_bias),
                                           static_cast<float*>(d_ws), static_cast<size_t>(ws_floats), sms,
                                           false);
        if (splits) *splits = sp;
        OPPO_CUDA_CHECK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
        return OPPO_OK;
    } catch (const oppo::Error& x) {
        oppo_set_global_error(x.what());
        return x.code;
    }
}

}  // extern "C"

// Times the engine GEMM alone: `copies` distinct weight matrices (a layer
// stack, so weights stream from HBM rather than L2), `reps` back-to-back
// launches on one stream bracketed by CUDA events.  avg_us = per launch.
extern "C" oppo_status oppo_k_gemm_bench(int32_t M, int32_t N, int32_t K, int32_t copies,
                                         int32_t reps, int32_t epilogue, float* avg_us) {
    try {
        cudaStream_t st;
        OPPO_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        __nv_bfloat16 *x = nullptr, *w = nullptr, *y = nullptr;
        const size_t wn = static_cast<size_t>(N) * K;
        OPPO_CUDA_CHECK(cudaMalloc(&x, static_cast<size_t>(M) * K * 2));
        OPPO_CUDA_CHECK(cudaMalloc(&w, wn * copies * 2));
        OPPO_CUDA_CHECK(cudaMalloc(&y, static_cast<size_t>(M) * N * 4));
        oppo::init_normal<__nv_bfloat16><<<(M * K + 255) / 256, 256, 0, st>>>(x, static_cast<int64_t>(M) * K, 1, 1, 1.0f);
        oppo::init_normal<__nv_bfloat16><<<static_cast<int>((wn * copies + 255) / 256), 256, 0, st>>>(
            w, static_cast<int64_t>(wn * copies), 1, 2, 0.02f);
        // LOGITS needs partials / keys: run through an EpiParams with real buffers
        float4* parts = nullptr;
        uint64_t* keys = nullptr;
        float* tl = nullptr;
        if (epilogue == oppo::EPI_LOGITS) {
            OPPO_CUDA_CHECK(cudaMalloc(&parts, static_cast<size_t>(M) * oppo::gemm_logit_tiles(OPPO_DTYPE_BF16, N) * 16));
            OPPO_CUDA_CHECK(cudaMalloc(&keys, static_cast<size_t>(M) * 8));
            OPPO_CUDA_CHECK(cudaMalloc(&tl, static_cast<size_t>(M) * 4));
            OPPO_CUDA_CHECK(cudaMemset(keys, 0x5a, static_cast<size_t>(M) * 8));
        }
        float* ws = nullptr;
        const size_t ws_floats = static_cast<size_t>(16) << 20;
        if (epilogue >= 16) OPPO_CUDA_CHECK(cudaMalloc(&ws, ws_floats * 4));
        __nv_bfloat16* aux = nullptr;  // SwiGLU backward: saved (gate, up) [M][2N]
        if (epilogue == oppo::EPI_SWIGLU_BWD) {
            OPPO_CUDA_CHECK(cudaMalloc(&aux, static_cast<size_t>(M) * 2 * N * 2));
            oppo::init_normal<__nv_bfloat16><<<static_cast<int>((static_cast<size_t>(M) * 2 * N + 255) / 256), 256, 0,
                                               st>>>(aux, static_cast<int64_t>(M) * 2 * N, 1, 3, 1.0f);
        }
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        auto launch = [&](int i) {
            if (epilogue >= 16) {  // decode GEMM, PDL-chained as inside the decode graph
                const int mode = epilogue - 16;
                oppo::gemm_dec_impl(nullptr, st, x, M, K, K, w + (i % copies) * wn, N, K, mode, y,
                                    mode == oppo::DEC_SWIGLU ? N / 2 : N, nullptr, ws, ws_floats, sms, true);
            } else if (epilogue == oppo::EPI_SWIGLU_BWD) {
                oppo::EpiParams ep{};
                ep.mode = oppo::EPI_SWIGLU_BWD;
                ep.y = y;
                ep.ldy = 2 * N;
                ep.aux = aux;
                oppo::gemm_with_params(OPPO_DTYPE_BF16, M, N, K, x, w + (i % copies) * wn, ep, st);
            } else if (epilogue == oppo::EPI_LOGITS) {
                oppo::EpiParams ep{};
                ep.mode = oppo::EPI_LOGITS;
                ep.partials = parts;
                ep.keys = keys;
                ep.tgt_logit = tl;
                oppo::gemm_with_params(OPPO_DTYPE_BF16, M, N, K, x, w + (i % copies) * wn, ep, st);
            } else {
                oppo::gemm_standalone(OPPO_DTYPE_BF16, M, N, K, x, w + (i % copies) * wn, nullptr, y,
                                      epilogue, st);
            }
        };
        for (int i = 0; i < 3; ++i) launch(i);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        OPPO_CUDA_CHECK(cudaEventRecord(a, st));
        for (int i = 0; i < reps; ++i) launch(i);
        OPPO_CUDA_CHECK(cudaEventRecord(b, st));
        OPPO_CUDA_CHECK(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        *avg_us = ms * 1e3f / reps;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaFree(x);
        cudaFree(w);
        cudaFree(y);
        if (parts) cudaFree(parts);
        if (keys) cudaFree(keys);
        if (tl) cudaFree(tl);
        if (ws) cudaFree(ws);
        if (aux) cudaFree(aux);
        cudaStreamDestroy(st);
        return OPPO_OK;
    } catch (const oppo::Error& x) {
        oppo_set_global_error(x.what());
        return x.code;
    }
}
