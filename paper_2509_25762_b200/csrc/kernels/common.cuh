// common.cuh — shared device helpers for the OPPO sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace oppo {

// ------------------------------------------------------------------ types
template <class T> struct Num;
template <> struct Num<float> {
    __device__ __forceinline__ static float to_f(float x) { return x; }
    __device__ __forceinline__ static float from_f(float x) { return x; }
};
template <> struct Num<__nv_bfloat16> {
    __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
    __device__ __forceinline__ static __nv_bfloat16 from_f(float x) { return __float2bfloat16(x); }
};
template <class T> __device__ __forceinline__ float tof(T x) { return Num<T>::to_f(x); }
template <class T> __device__ __forceinline__ T fromf(float x) { return Num<T>::from_f(x); }

// ---------------------------------------------------------------- hashing
// Counter-based streams used for weights, prompts and sampling noise.  The
// same integer arithmetic is restated in oracle/oppo_oracle.c.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}
// per-(sequence, response position) key of the sampling stream
__host__ __device__ __forceinline__ uint64_t token_key(uint64_t seed, int64_t seq_id, int32_t pos) {
    return mix64(seed ^ mix64(static_cast<uint64_t>(seq_id) * 0x100000001b3ull +
                              static_cast<uint64_t>(static_cast<uint32_t>(pos))));
}
// uniform in (0,1) for vocabulary entry v under a token key
__host__ __device__ __forceinline__ float key_uniform(uint64_t key, uint32_t v) {
    uint32_t x = static_cast<uint32_t>(key) ^ (v * 0x9e3779b9u);
    x = lowbias32(x) ^ static_cast<uint32_t>(key >> 32);
    x = lowbias32(x);
    // 23 random bits: the largest value, 1 - 2^-24, is exactly representable (24 bits
    // would round up to 1.0f and give an infinite Gumbel draw)
    return (static_cast<float>(x >> 9) + 0.5f) * (1.0f / 8388608.0f);
}
__device__ __forceinline__ float gumbel_noise(uint64_t key, uint32_t v) {
    return -logf(-logf(key_uniform(key, v)));
}

// Two-level sampling streams (see gemm.cuh logits_tile / model.cuh logits_combine):
// vocabulary blocks of kSampleBlock ids, per-block Gumbel noise and in-block uniform.
constexpr int kSampleBlock = 256;
constexpr uint64_t kInBlockKey = 0x696e626c6f636bull;  // "inblock"
constexpr uint64_t kBlockKey = 0x626c6f636b6e7a65ull;  // "blocknze"

// Programmatic dependent launch: let the next kernel in the stream start its
// prologue now / wait until the previous kernel's results are visible.  Both
// are no-ops when the kernel was launched without the PDL attribute.
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ------------------------------------------------------------ reductions
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// 16-byte vector of T
template <class T> struct Vec16 {
    static constexpr int N = 16 / sizeof(T);
};

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

// Paged KV cache view: per model and layer, K and V pools of pages laid out
// [page][kv_head][page_size][head_dim]; a slot's page table maps position -> page.
struct KvView {
    void* k;              // pool base of layer 0
    void* v;
    int64_t layer_stride; // elements between layers
    int32_t page_size;
    int32_t kv_heads;
    int32_t head_dim;
    const int32_t* page_table;  // [slots][max_pages]
    int32_t max_pages;
};

template <class T>
__device__ __forceinline__ size_t kv_index(const KvView& kv, int layer, int slot, int pos, int h) {
    const int page = kv.page_table[slot * kv.max_pages + pos / kv.page_size];
    return static_cast<size_t>(layer) * kv.layer_stride +
           ((static_cast<size_t>(page) * kv.kv_heads + h) * kv.page_size + pos % kv.page_size) *
               kv.head_dim;
}

}  // namespace oppo

#define OPPO_CUDA_CHECK(expr)                                                          \
    do {                                                                               \
        cudaError_t _e = (expr);                                                       \
        if (_e != cudaSuccess)                                                         \
            throw ::oppo::Error(OPPO_ERR_CUDA, std::string(#expr) + ": " +             \
                                                   cudaGetErrorString(_e));            \
    } while (0)
