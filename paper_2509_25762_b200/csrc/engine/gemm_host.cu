// gemm_host.cu — host launcher of the engine GEMM: TMA descriptors (cached),
// token-tile (UMMA_N) selection and split-K sizing.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "engine.cuh"
#include "kernels/gemm.cuh"
#include "kernels/gemm_dec.cuh"
#include "kernels/lmhead_dec.cuh"

namespace oppo {

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw Error(OPPO_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

template <int BN>
void launch_tc(const CUtensorMap& mx, const CUtensorMap& mw, dim3 grid, const GemmShape& sh,
               const EpiParams& ep, cudaStream_t st, bool pdl) {
    static std::once_flag attr;
    std::call_once(attr, [] {
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(tc::gemm_bf16_tc<BN>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             tc::Cfg<BN>::SMEM));
    });
    launch(pdl, tc::gemm_bf16_tc<BN>, grid, dim3(128), tc::Cfg<BN>::SMEM, st, mx, mw, sh, ep);
}
}  // namespace

// K-major 2D map over a [rows, cols] matrix with leading dimension ld
// (elements), box = [box_rows, 64], 128B swizzle, zero fill out of bounds.
CUtensorMap make_tma_2d(const void* ptr, int rows, int cols, int ld, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr),
                                   dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw Error(OPPO_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return m;
}

static const CUtensorMap& cached_map(Engine* e, const void* ptr, int rows, int cols, int ld,
                                     int box_rows, CUtensorMap& scratch) {
    if (!e) {
        scratch = make_tma_2d(ptr, rows, cols, ld, box_rows);
        return scratch;
    }
    const TmaKey k{ptr, rows, cols, box_rows, ld};
    std::lock_guard<std::mutex> lk(e->tma_mu);  // std::map nodes stay put: the reference outlives the lock
    auto it = e->tma_cache.find(k);
    if (it == e->tma_cache.end())
        it = e->tma_cache.emplace(k, make_tma_2d(ptr, rows, cols, ld, box_rows)).first;
    return it->second;
}

const CUtensorMap& cached_map_pub(Engine* e, const void* ptr, int rows, int cols, int ld, int box_rows,
                                  CUtensorMap& scratch) {
    return cached_map(e, ptr, rows, cols, ld, box_rows, scratch);
}

int gemm_logit_tiles(int, int N) { return (N + kSampleBlock - 1) / kSampleBlock; }

// x: [M, K] (ld ldx), w: [N, K] (ld ldw).  bf16: 128-token tiles (A operand,
// zero-filled past M by TMA) x BN-row weight tiles; BN = 256 for prefill and
// the lm_head, 64/128 for decode so the grid covers the SMs; split-K when the
// tile count is still under half the SMs.
int persist_mode() {  // read per call so tests can compare both kernels in one process
    const char* v = std::getenv("OPPO_GEMM_PERSIST");
    return v ? std::atoi(v) : 0;  // 0 off (slower in the cfg2 bench), 1 everywhere, 2 PPO update only
}
bool tc2sm_long_enabled() {  // read per call so tests can compare both kernels in one process
    const char* v = std::getenv("OPPO_TC2SM_LONGK");
    return v ? std::atoi(v) != 0 : true;  // measured: update 912 -> 887 ms at 39K tokens
}
bool raster_n_fast() {  // read per call (A/B in one process)
    const char* v = std::getenv("OPPO_RASTER_N");
    return v ? std::atoi(v) != 0 : true;
}
bool tc2sm_short_enabled() {  // read per call (A/B in one process)
    const char* v = std::getenv("OPPO_TC2SM_SHORT");
    return v ? std::atoi(v) != 0 : false;
}
// cost-model latency (ns) of one fold round trip in the consuming kernel
static const double g_fold_ns = [] {
    const char* v = std::getenv("OPPO_DEC_FOLD_NS");
    return v ? std::atof(v) : 400.0;  // measured: -8% decode iteration at 16 rows, neutral above
}();


static void gemm_impl(Engine* e, Work* wk, cudaStream_t st, const void* x, int M, int K, int ldx,
                      const void* wt, int N, int ldw, const EpiParams& ep_in, int dtype,
                      int num_sms, float* ws, size_t ws_floats, int* cnt, int cnt_n, int a_mn = 0,
                      int b_mn = 0) {
    if (M <= 0 || N <= 0) return;
    EpiParams ep = ep_in;
    ep.M = M;
    ep.N = N;
    ep.n_tiles = gemm_logit_tiles(dtype, N);
    GemmShape sh{M, N, K, 1, 0, nullptr, nullptr, a_mn, b_mn, ldx, ldw};
    const int m_tiles = (M + 127) / 128;
    const bool rope = ep.mode == EPI_ROPE_APPEND;
    const bool mn = a_mn || b_mn;
    if (rope && (dtype != OPPO_DTYPE_BF16 || (ep.kv.head_dim != 64 && ep.kv.head_dim != 128)))
        throw Error(OPPO_ERR_INTERNAL, "rope-append epilogue: bf16, head_dim 64 or 128 only");
    if (mn && (ep.mode == EPI_LOGITS || rope))
        throw Error(OPPO_ERR_INTERNAL, "MN-major operands: store / add / softmax-grad epilogues only");
    if (dtype == OPPO_DTYPE_F32) {
        launch(e && e->pdl, gemm_simt<float>, dim3(m_tiles, (N + kSampleBlock - 1) / kSampleBlock),
               dim3(128), 0, st, static_cast<const float*>(x), static_cast<const float*>(wt), sh, ep);
        OPPO_CUDA_CHECK(cudaGetLastError());
        return;
    }
    // Token-rich prefill GEMMs (>= 8 token tiles, not the logits epilogue):
    // persistent kernel, one CTA per SM, 192 KB TMA ring, double-buffered TMEM
    // (OPPO_GEMM_PERSIST=1; measured: qkv 28.8 -> 22.7 us, gate|up 183 -> 172 us
    // at 8192 rows alone, but the cfg2 bench loses 1% with it: 212.2 -> 210.1)
    // Epilogue-light modes only: with a residual read-modify-write or the
    // transposed softmax-grad stores, the 4 epilogue warps fall behind the
    // mainloop and the 2-CTA/SM kernel (8 epilogue warps per SM) wins
    // (bench: update 60 -> 69 ms on the persistent kernel; O / down no gain).
    const bool light = ep.mode == EPI_STORE || ep.mode == EPI_SWIGLU || ep.mode == EPI_ROPE_APPEND;
    const int pm = persist_mode();
    // (2: the update's GEMMs with any epilogue but the logits one, K-major or MN-major operands)
    // (long-K gradient GEMMs stay on the CTA-pair kernel below)
    const bool pair_long = ep.pair_long_k && tc2sm_long_enabled() && (K + 63) / 64 >= 64;
    const bool persist = dtype == OPPO_DTYPE_BF16 && m_tiles >= 8 &&
                         ((pm == 1 && light && !mn) ||
                          (pm == 2 && ep.update_gemm && ep.mode != EPI_LOGITS && !pair_long));
    if (persist) {
        // 128-wide tiles where a 256-wide last tile would waste > 5% (N = 896, 1152)
        const int pad256 = (N + 255) / 256 * 256 - N;
        const int BNp = (N % 128 == 0 && pad256 * 20 > N) ? 128 : 256;
        sh.splits = 1;
        sh.kb_per_split = (K + 63) / 64;
        sh.n_fast = raster_n_fast();
        CUtensorMap s1, s2;
        const CUtensorMap& mx = a_mn ? cached_map(e, x, K, M, ldx, 64, s1) : cached_map(e, x, M, K, ldx, 128, s1);
        const CUtensorMap& mw = b_mn ? cached_map(e, wt, K, N, ldw, 64, s2) : cached_map(e, wt, N, K, ldw, BNp, s2);
        const int total = m_tiles * ((N + BNp - 1) / BNp);
        const dim3 grid(std::min(total, num_sms));
        if (BNp == 256) {
            static std::once_flag a256;
            std::call_once(a256, [] {
                OPPO_CUDA_CHECK(cudaFuncSetAttribute(tc::gemm_bf16_persist<256>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     tc::CfgP<256>::SMEM));
            });
            launch(e && e->pdl, tc::gemm_bf16_persist<256>, grid, dim3(tc::kPersistThreads), tc::CfgP<256>::SMEM, st,
                   mx, mw, sh, ep);
        } else {
            static std::once_flag a128;
            std::call_once(a128, [] {
                OPPO_CUDA_CHECK(cudaFuncSetAttribute(tc::gemm_bf16_persist<128>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     tc::CfgP<128>::SMEM));
            });
            launch(e && e->pdl, tc::gemm_bf16_persist<128>, grid, dim3(tc::kPersistThreads), tc::CfgP<128>::SMEM, st,
                   mx, mw, sh, ep);
        }
        OPPO_CUDA_CHECK(cudaGetLastError());
        return;
    }
    // Token-rich prefill GEMMs: CTA-pair 256x256 tiles (cta_group::2)
    // (not on the scorer streams: cluster launches inside the scorer's green
    // context hung in round-1 measurements, so prefill keeps single-CTA tiles)
    const bool scorer_stream = e && (st == e->ss || st == e->ss_m[0] || st == e->ss_m[1]);
    // Long-K GEMMs that fill the GPU with CTA pairs (the update's weight
    // gradients, K = tokens): the pair tile halves each SM's operand stream
    // per flop, and the 6-stage ring covers the L2 latency (OPPO_TC2SM_LONGK)
    const int kb_all = (K + 63) / 64;
    const int pairs = ((m_tiles + 1) / 2) * ((N + 255) / 256);
    const bool long2 = ep.pair_long_k && tc2sm_long_enabled() && !scorer_stream && kb_all >= 64 && m_tiles >= 2 &&
                       pairs * 2 * 10 >= num_sms * 9 && ep.mode != EPI_LOGITS && !rope;
    // the update's token-rich short-K GEMMs (forward, dgrad against D-wide
    // weights) on CTA pairs, two pairs per SM pair (OPPO_TC2SM_SHORT)
    const bool short2 = ep.update_gemm && tc2sm_short_enabled() && !long2 && m_tiles >= 8 && N >= 512 &&
                        pairs * 2 >= num_sms && ep.mode != EPI_LOGITS && !rope;
    if (long2 || short2) {
        static std::once_flag attr2;
        std::call_once(attr2, [] {
            OPPO_CUDA_CHECK(cudaFuncSetAttribute(tc::gemm_bf16_tc2sm<6>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 tc::Cfg2Sm<6>::SMEM));
            OPPO_CUDA_CHECK(cudaFuncSetAttribute(tc::gemm_bf16_tc2sm<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 tc::Cfg2Sm<3>::SMEM));
        });
        sh.splits = 1;
        sh.kb_per_split = (K + 63) / 64;
        CUtensorMap s1, s2;
        const CUtensorMap& mx = a_mn ? cached_map(e, x, K, M, ldx, 64, s1) : cached_map(e, x, M, K, ldx, 128, s1);
        const CUtensorMap& mw = b_mn ? cached_map(e, wt, K, N, ldw, 64, s2) : cached_map(e, wt, N, K, ldw, 128, s2);
        const int mt2 = (m_tiles + 1) / 2 * 2;  // whole CTA pairs (OOB rows zero-filled)
        sh.n_fast = raster_n_fast();
        const dim3 grid2 = sh.n_fast ? dim3(2 * ((N + 255) / 256), mt2 / 2) : dim3(mt2, (N + 255) / 256);
        const dim3 clu(2, 1, 1);
        if (long2)
            launch_cluster(e && e->pdl, clu, tc::gemm_bf16_tc2sm<6>, grid2, dim3(128), tc::Cfg2Sm<6>::SMEM, st, mx, mw,
                           sh, ep);
        else
            launch_cluster(e && e->pdl, clu, tc::gemm_bf16_tc2sm<3>, grid2, dim3(128), tc::Cfg2Sm<3>::SMEM, st, mx, mw,
                           sh, ep);
        OPPO_CUDA_CHECK(cudaGetLastError());
        return;
    }
    // Token-rich (prefill) GEMMs use 128x256 tiles.  Decode GEMMs (a few token
    // tiles) are weight-streaming: pick the widest weight tile that still gives
    // ~one CTA per SM, then split K (at most 4 ways, so the deterministic
    // last-arriver fixup stays small) until the grid covers the SMs.
    int BN;
    // prefill: 128x256 tiles, except narrow outputs (N <= 1024: the O and down
    // projections) of mid-size passes, where 128x128 tiles double the CTAs
    // (measured at 2048 rows: down 58.9 -> 34.7 us, O 24.6 -> 16.4 us; at
    // 8192 rows 256 stays ahead; the cfg2 bench prefers the cut at 2048).
    // OPPO_PREFILL_NARROW_ROWS moves the cut.
    static const int narrow_rows = [] {
        const char* v = std::getenv("OPPO_PREFILL_NARROW_ROWS");
        return v ? std::atoi(v) : 2048;  // bench sweep 1024/2048/4096/8192: 2048 best by ~0.3%
    }();
    if (ep.mode == EPI_LOGITS || m_tiles > 4) {
        static const int wide_m = [] {  // vocabulary-row GEMMs (the update's dW): M >= this -> 128-wide
            const char* v = std::getenv("OPPO_NARROW_WIDE_M");
            return v ? std::atoi(v) : 0;
        }();
        BN = (ep.mode != EPI_LOGITS && N <= 1024 && (M <= narrow_rows || (wide_m > 0 && M >= wide_m))) ? 128 : 256;
    } else {
        BN = 64;
        for (int b : {256, 128})
            if (m_tiles * ((N + b - 1) / b) >= num_sms) {
                BN = b;
                break;
            }
    }
    if (rope && BN < ep.kv.head_dim) BN = ep.kv.head_dim;  // whole heads per tile
    const int n_tiles = (N + BN - 1) / BN;
    const int kb = (K + 63) / 64;
    const int tiles = n_tiles * m_tiles;
    int splits = 1;
    // long-K GEMMs with few output tiles (the update's weight gradients, K =
    // tokens; its vocabulary dgrad, K = V): split K until both CTA slots of
    // every SM are busy (133 tiles of dW_down ran at 45% of the slots)
    const bool long_k = m_tiles > 4 && kb >= 64 && !(e && (st == e->ss || st == e->ss_m[0] || st == e->ss_m[1]));
    if (ws && cnt && ep.mode != EPI_LOGITS && long_k && tiles * 4 <= 3 * 2 * num_sms) {
        splits = std::max(1, std::min((2 * num_sms) / tiles, 8));
        while (splits > 1 && (static_cast<size_t>(splits) * tiles * 128 * BN > ws_floats || tiles > cnt_n))
            --splits;
    } else if (ws && cnt && ep.mode != EPI_LOGITS && tiles * 2 <= num_sms && kb >= 4) {
        splits = std::max(1, std::min(std::min(kb / 2, (num_sms + tiles - 1) / tiles), 4));
        while (splits > 1 && (static_cast<size_t>(splits) * tiles * 128 * BN > ws_floats ||
                              tiles > cnt_n))
            --splits;
    }
    const int kbps = (kb + splits - 1) / splits;
    splits = (kb + kbps - 1) / kbps;
    sh.splits = splits;
    sh.kb_per_split = kbps;
    sh.workspace = ws;
    sh.counters = cnt;
    CUtensorMap s1, s2;
    // MN-major operands are stored [K][M] / [K][N]: [64 k][64] boxes
    const CUtensorMap& mx = a_mn ? cached_map(e, x, K, M, ldx, 64, s1) : cached_map(e, x, M, K, ldx, 128, s1);
    const CUtensorMap& mw = b_mn ? cached_map(e, wt, K, N, ldw, 64, s2) : cached_map(e, wt, N, K, ldw, BN, s2);
    // token-rich GEMMs: feature tiles fastest, so the CTAs reading one token
    // tile run together (a 32K-row update GEMM re-read its 59 MB token operand
    // from DRAM once per feature tile with the m-fast order: 1.57 GB read by
    // the SwiGLU-backward GEMM for 0.64 GB of algorithmic reads)
    sh.n_fast = m_tiles >= 8 && raster_n_fast();
    const dim3 grid = sh.n_fast ? dim3(n_tiles, m_tiles, splits) : dim3(m_tiles, n_tiles, splits);
    switch (BN) {
    case 64:
        launch_tc<64>(mx, mw, grid, sh, ep, st, e && e->pdl);
        break;
    case 128:
        launch_tc<128>(mx, mw, grid, sh, ep, st, e && e->pdl);
        break;
    default:
        launch_tc<256>(mx, mw, grid, sh, ep, st, e && e->pdl);
        break;
    }
    OPPO_CUDA_CHECK(cudaGetLastError());
    (void)wk;
}

// Decode-shaped GEMM (swap-AB, gemm_dec.cuh).  Chooses the token grouping,
// the K split and the pipeline depth; returns the number of K splits whose
// fp32 partials the consumer must fold (DEC_PARTIAL), 1 otherwise.
// Split choice: minimise (waves x per-CTA stage bytes / per-SM TMA ingest)
// + (partials written and re-read through L2), subject to the workspace.
int gemm_dec_impl(Engine* e, cudaStream_t st, const void* x, int M, int K, int ldx, const void* wt,
                  int N, int ldw, int mode, void* y, int ldy, const float* bias, float* ws,
                  size_t ws_floats, int num_sms, bool pdl) {
    if (M <= 0 || N <= 0) return 1;
    const int Mp = (M + 15) / 16 * 16;
    if (Mp > 512 || K % 64 != 0) throw Error(OPPO_ERR_INTERNAL, "gemm_dec shape out of range");
    DecShape s{};
    s.M = M;
    s.N = N;
    s.K = K;
    s.nbox = Mp > 256 ? 2 : 1;
    s.box_rows = ((Mp + s.nbox - 1) / s.nbox + 15) / 16 * 16;
    const int stage = dec::kWBytes + s.nbox * s.box_rows * 128;
    const int kb_total = K / 64;
    const int tiles = (N + 127) / 128;
    int splits = 1;
    if (mode == DEC_PARTIAL) {
        double best = 1e30;
        for (int sp = 1; sp <= std::min(kb_total, 64); ++sp) {
            const int kbps = (kb_total + sp - 1) / sp;
            const int se = (kb_total + kbps - 1) / kbps;
            if (static_cast<size_t>(se) * M * N > ws_floats) break;
            const int waves = (tiles * se + num_sms - 1) / num_sms;
            // + the consumer's fold: one dependent L2 round trip per 8 splits
            const double t = waves * (kbps * static_cast<double>(stage) / 60.0) +
                             se * static_cast<double>(M) * N * 8.0 / 8000.0 + ((se + 7) / 8) * g_fold_ns;
            if (t < best - 1e-9) {
                best = t;
                splits = se;
            }
        }
    }
    s.kb_per_split = (kb_total + splits - 1) / splits;
    splits = (kb_total + s.kb_per_split - 1) / s.kb_per_split;
    s.stages = std::max(1, std::min(s.kb_per_split, std::min(8, (200 * 1024) / stage)));
    int cols = 32;
    while (cols < (s.nbox == 2 ? 512 : s.box_rows)) cols *= 2;
    s.tmem_cols = cols;
    s.mode = mode;
    s.y = y;
    s.ldy = ldy;
    s.bias = bias;
    s.ws = ws;
    const int smem = s.stages * stage + 1024 + 256;
    static std::once_flag attr;
    std::call_once(attr, [] {
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(dec::gemm_dec, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024));
    });
    CUtensorMap s1, s2;
    const CUtensorMap& mw = cached_map(e, wt, N, K, ldw, 128, s1);
    const CUtensorMap& mx = cached_map(e, x, M, K, ldx, s.box_rows, s2);
    launch(pdl, dec::gemm_dec, dim3(tiles, splits), dim3(128), smem, st, mw, mx, s);
    OPPO_CUDA_CHECK(cudaGetLastError());
    return mode == DEC_PARTIAL ? splits : 1;
}

// Decode lm_head + in-block sampling (lmhead_dec.cuh), <= 128 tokens.
void lmhead_dec_run(Engine& e, Work& w, cudaStream_t st, const void* x, int M, int K, const void* wt,
                    int V, float4* partials, const uint64_t* keys) {
    lmh::Shape s{};
    s.M = M;
    s.Mp = (M + 15) / 16 * 16;
    s.N = V;
    s.K = K;
    const int stage = lmh::kWBytes + s.Mp * 128;
    s.stages = std::max(1, std::min(K / 64, (200 * 1024) / stage));
    int cols = 32;
    while (cols < 2 * s.Mp) cols *= 2;
    s.tmem_cols = cols;
    s.n_tiles = gemm_logit_tiles(OPPO_DTYPE_BF16, V);
    s.partials = partials;
    s.keys = keys;
    const int smem = s.stages * stage + 1024 + 2048;
    static std::once_flag attr;
    std::call_once(attr, [] {
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(lmh::lmhead_dec, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024));
    });
    CUtensorMap s1, s2;
    const CUtensorMap& mw = cached_map(&e, wt, V, K, K, 256, s1);
    const CUtensorMap& mx = cached_map(&e, x, M, K, K, s.Mp, s2);
    launch(e.pdl, lmh::lmhead_dec, dim3((V + 255) / 256), dim3(128), smem, st, mw, mx, s);
    OPPO_CUDA_CHECK(cudaGetLastError());
    e.launches += 1;
    (void)w;
}

int gemm_dec_run(Engine& e, Work& w, cudaStream_t st, const void* x, int M, int K, int ldx,
                 const void* wt, int N, int ldw, int mode, void* y, int ldy, const float* bias) {
    e.launches += 1;
    return gemm_dec_impl(&e, st, x, M, K, ldx, wt, N, ldw, mode, y, ldy, bias, w.gemm_ws,
                         w.gemm_ws_floats, w.sms, e.pdl);
}

void gemm_run(Engine& e, Work& w, cudaStream_t st, const void* x, int M, int K, int ldx,
              const void* wt, int N, int ldw, const EpiParams& ep) {
    gemm_impl(&e, &w, st, x, M, K, ldx, wt, N, ldw, ep, e.dtype, w.sms, w.gemm_ws,
              w.gemm_ws_floats, w.gemm_cnt, w.gemm_cnt_n);
    e.launches += 1;
}

void gemm_run_t(Engine& e, Work& w, cudaStream_t st, const void* a, int a_mn, int lda, const void* b, int b_mn,
                int ldb, int M, int N, int K, const EpiParams& ep) {
    gemm_impl(&e, &w, st, a, M, K, lda, b, N, ldb, ep, e.dtype, w.sms, w.gemm_ws, w.gemm_ws_floats, w.gemm_cnt,
              w.gemm_cnt_n, a_mn, b_mn);
    e.launches += 1;
}

void gemm_standalone_t(int dtype, int M, int N, int K, const void* a, int a_mn, int lda, const void* b, int b_mn,
                       int ldb, void* y, int epi, cudaStream_t st) {
    EpiParams ep{};
    ep.pair_long_k = 1;  // as the update's GEMMs
    ep.update_gemm = 1;
    ep.mode = epi;
    ep.y = y;
    ep.ldy = N;
    ep.scale = 1.0f;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    gemm_impl(nullptr, nullptr, st, a, M, K, lda, b, N, ldb, ep, dtype, sms, nullptr, 0, nullptr, 0, a_mn, b_mn);
}

void gemm_standalone(int dtype, int M, int N, int K, const void* x, const void* w,
                     const float* bias, void* y, int epi, cudaStream_t st) {
    EpiParams ep{};
    ep.mode = epi;
    ep.y = y;
    ep.ldy = epi == EPI_SWIGLU ? N / 2 : N;
    ep.bias = bias;
    ep.scale = 1.0f;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    gemm_impl(nullptr, nullptr, st, x, M, K, K, w, N, K, ep, dtype, sms, nullptr, 0, nullptr, 0);
}

void gemm_with_params(int dtype, int M, int N, int K, const void* x, const void* w,
                      const EpiParams& ep, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    gemm_impl(nullptr, nullptr, st, x, M, K, K, w, N, K, ep, dtype, sms, nullptr, 0, nullptr, 0);
}

}  // namespace oppo

// ------------------------------------------------------------------------
// TMA streaming probe (perf diagnosis, tools/tma_probe.py): each CTA streams
// `tiles` boxes of [box_rows x 64] bf16 from a row-major matrix through a ring
// of `stages` shared-memory buffers with mbarrier completion, no compute.
namespace oppo {
namespace probe {
__global__ void __launch_bounds__(32) tma_stream(const __grid_constant__ CUtensorMap map, int rows, int kb_total,
                                                 int per_cta, int stages, int box_bytes, unsigned* sink) {
    extern __shared__ uint8_t sm_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + stages * box_bytes);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) tc::mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    const int row_tiles = rows / (box_bytes / 128);
    uint32_t phase = 0;
    int issued = 0, done = 0;
    const int first = blockIdx.x * per_cta;
    auto issue = [&](int t) {
        const int s = t % stages;
        const int g = first + t;
        const int rt = g % row_tiles, kb = (g / row_tiles) % kb_total;
        tc::mbar_expect_tx(&full[s], box_bytes);
        tc::tma_load_2d(sm + s * box_bytes, &map, &full[s], kb * 64, rt * (box_bytes / 128));
    };
    for (; issued < stages && issued < per_cta; ++issued) issue(issued);
    for (; done < per_cta; ++done) {
        const int s = done % stages;
        tc::mbar_wait(&full[s], (done / stages) & 1);
        if (issued < per_cta) issue(issued++);
    }
    (void)phase;
    if (blockIdx.x == 0) *sink = sm[7];
}
}  // namespace probe
}  // namespace oppo

extern "C" oppo_status oppo_k_tma_probe(int32_t ctas, int32_t stages, int32_t box_rows, int32_t per_cta,
                                        float* us, float* gbs) {
    try {
        const int K = 4096, rows = 16384;  // 128 MB bf16 matrix (> L2)
        void* buf = nullptr;
        unsigned* sink = nullptr;
        OPPO_CUDA_CHECK(cudaMalloc(&buf, static_cast<size_t>(rows) * K * 2));
        OPPO_CUDA_CHECK(cudaMalloc(&sink, 64));
        OPPO_CUDA_CHECK(cudaMemset(buf, 0, static_cast<size_t>(rows) * K * 2));
        const CUtensorMap m = oppo::make_tma_2d(buf, rows, K, K, box_rows);
        const int box_bytes = box_rows * 128;
        const int smem = stages * box_bytes + 1024 + 256;
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(oppo::probe::tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int w = 0; w < 2; ++w)
            oppo::probe::tma_stream<<<ctas, 32, smem>>>(m, rows, K / 64, per_cta, stages, box_bytes, sink);
        cudaEventRecord(a);
        const int reps = 5;
        for (int r = 0; r < reps; ++r)
            oppo::probe::tma_stream<<<ctas, 32, smem>>>(m, rows, K / 64, per_cta, stages, box_bytes, sink);
        cudaEventRecord(b);
        OPPO_CUDA_CHECK(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        *us = ms * 1e3f / reps;
        *gbs = static_cast<float>(static_cast<double>(ctas) * per_cta * box_bytes / (*us * 1e-6) / 1e9);
        cudaFree(buf);
        cudaFree(sink);
        return OPPO_OK;
    } catch (const oppo::Error& x) {
        oppo_set_global_error(x.what());
        return x.code;
    }
}
