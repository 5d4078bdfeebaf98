// gemm_host.cu — host launcher of the engine GEMM: TMA descriptors (cached),
// token-tile (UMMA_N) selection and split-K sizing.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "engine.cuh"
#include "kernels/gemm.cuh"

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
void launch_tc(const CUtensorMap& mw, const CUtensorMap& mx, dim3 grid, const GemmShape& sh,
               const EpiParams& ep, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        OPPO_CUDA_CHECK(cudaFuncSetAttribute(tc::gemm_bf16_tc<BN>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             tc::Cfg<BN>::SMEM));
        attr = true;
    }
    tc::gemm_bf16_tc<BN><<<grid, 128, tc::Cfg<BN>::SMEM, st>>>(mw, mx, sh, ep);
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
    auto it = e->tma_cache.find(k);
    if (it == e->tma_cache.end())
        it = e->tma_cache.emplace(k, make_tma_2d(ptr, rows, cols, ld, box_rows)).first;
    return it->second;
}

// x: [M, K] (ld ldx), w: [N, K] (ld ldw).  For bf16 the token rows of the
// TMA map span the whole workspace (w.max_rows) so the cached descriptor is
// reused across iterations; rows >= M only feed masked output columns.
static void gemm_impl(Engine* e, Work* wk, cudaStream_t st, const void* x, int M, int K, int ldx,
                      const void* wt, int N, int ldw, const EpiParams& ep_in, int dtype,
                      int num_sms, float* ws, size_t ws_floats, int* cnt, int cnt_n) {
    if (M <= 0 || N <= 0) return;
    EpiParams ep = ep_in;
    ep.M = M;
    ep.N = N;
    GemmShape sh{M, N, K, 1, 0, nullptr, nullptr, 32};
    if (dtype == OPPO_DTYPE_F32) {
        ep.n_tiles = (N + 127) / 128;
        dim3 grid((N + 127) / 128, (M + 31) / 32);
        if (ldx != K || ldw != K) throw Error(OPPO_ERR_INTERNAL, "SIMT GEMM needs packed rows");
        gemm_simt<float><<<grid, 128, 0, st>>>(static_cast<const float*>(x),
                                               static_cast<const float*>(wt), sh, ep);
        OPPO_CUDA_CHECK(cudaGetLastError());
        return;
    }
    // token tile: UMMA_N = bn (multiple of 16, <= 256)
    const int m_tiles = (M + 255) / 256;
    int bn = (M + m_tiles - 1) / m_tiles;
    bn = (bn + 15) / 16 * 16;
    int BN = 32;
    while (BN < bn) BN *= 2;
    const int n_tiles = (N + 127) / 128;
    ep.n_tiles = n_tiles;
    const int kb = (K + 63) / 64;
    const int tiles = n_tiles * m_tiles;
    int splits = 1;
    if (ws && cnt && tiles * 2 <= num_sms && kb >= 8) {
        splits = std::min(kb / 4, (num_sms + tiles - 1) / tiles);
        splits = std::max(1, splits);
        const size_t need = static_cast<size_t>(splits) * tiles * 128 * BN;
        while (splits > 1 && (static_cast<size_t>(splits) * tiles * 128 * BN > ws_floats ||
                              tiles > cnt_n))
            --splits;
        (void)need;
    }
    const int kbps = (kb + splits - 1) / splits;
    splits = (kb + kbps - 1) / kbps;
    sh.splits = splits;
    sh.kb_per_split = kbps;
    sh.workspace = ws;
    sh.counters = cnt;
    sh.bn = bn;
    const int x_rows = wk ? std::max(wk->max_rows, M) : M;
    CUtensorMap s1, s2;
    const CUtensorMap& mw = cached_map(e, wt, N, K, ldw, 128, s1);
    const CUtensorMap& mx = cached_map(wk ? e : nullptr, x, x_rows, K, ldx, bn, s2);
    dim3 grid(n_tiles, m_tiles, splits);
    (void)BN;
    // the runtime UMMA_N is bn; BN picks the TMEM allocation / smem carve-out
    switch (BN) {
    case 32:
        launch_tc<32>(mw, mx, grid, sh, ep, st);
        break;
    case 64:
        launch_tc<64>(mw, mx, grid, sh, ep, st);
        break;
    case 128:
        launch_tc<128>(mw, mx, grid, sh, ep, st);
        break;
    default:
        launch_tc<256>(mw, mx, grid, sh, ep, st);
        break;
    }
    OPPO_CUDA_CHECK(cudaGetLastError());
}

void gemm_run(Engine& e, Work& w, cudaStream_t st, const void* x, int M, int K, int ldx,
              const void* wt, int N, int ldw, const EpiParams& ep) {
    gemm_impl(&e, &w, st, x, M, K, ldx, wt, N, ldw, ep, e.dtype, e.num_sms, w.gemm_ws,
              w.gemm_ws_floats, w.gemm_cnt, w.gemm_cnt_n);
    e.launches += 1;
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

}  // namespace oppo
