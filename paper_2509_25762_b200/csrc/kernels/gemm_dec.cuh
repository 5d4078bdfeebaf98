// gemm_dec.cuh — decode-shaped GEMM Y[M,N] = X[M,K] . W[N,K]^T for a few
// hundred tokens (M <= 512), the actor's per-iteration projections.
//
// Swap-AB on tcgen05: the WEIGHT tile is the UMMA A operand (128 weight rows
// on the 128 TMEM lanes) and the tokens are the UMMA N dimension (16..256 per
// MMA, two MMA groups above 256 tokens), so shared memory holds only the
// tokens that exist (no 128-row zero-filled activation tile) and every CTA
// streams a disjoint 128-row x (K / splits) slab of W from HBM.
//   - grid = (N / 128 weight tiles, K splits), one CTA per SM (deep TMA
//     pipeline, up to ~200 KB of stages); W stages are issued before the PDL
//     wait, so weights stream while the previous kernel drains.
//   - epilogue: thread = TMEM lane = weight row n, 16 tokens per tcgen05.ld;
//     stores are warp-coalesced along n.
//   - DEC_PARTIAL writes this split's fp32 partial sums to ws[split][m][n];
//     the CONSUMER kernel (RMSNorm residual add, RoPE/KV append) folds the
//     splits in a fixed order, so there are no counters, no atomics and the
//     result is deterministic.  DEC_SWIGLU (unsplit) applies silu(g)*u to the
//     interleaved (gate_i, up_i) row pairs of adjacent lanes.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "common.cuh"
#include "gemm.cuh"

namespace oppo {

enum DecMode : int { DEC_PARTIAL = 0, DEC_SWIGLU = 1, DEC_STORE = 2 };

struct DecShape {
    int M, N, K;        // tokens, weight rows (outputs), reduction
    int nbox;           // token groups per stage (1, or 2 above 256 tokens)
    int box_rows;       // tokens per group (multiple of 16, <= 256)
    int kb_per_split;   // 64-wide k blocks per split
    int stages;
    int tmem_cols;      // power of two >= 32
    int mode;           // DecMode
    void* y;            // DEC_SWIGLU / DEC_STORE output (bf16), row stride ldy
    int ldy;
    const float* bias;  // DEC_STORE only
    float* ws;          // DEC_PARTIAL: [split][M][N] fp32
};

namespace dec {

constexpr int kWBytes = 128 * 64 * 2;  // one 128-row x 64-k weight tile

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// kind::f16: D=f32, A=B=bf16, both K-major; N = token group, M = 128 weight rows
__device__ __forceinline__ uint32_t idesc(int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(128 >> 4) << 24);
}

static __global__ void __launch_bounds__(128, 1)
    gemm_dec(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
             DecShape s) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int XB = s.box_rows * 128;
    const int STAGE = kWBytes + s.nbox * XB;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + s.stages * STAGE);
    uint64_t* empty = full + s.stages;
    uint64_t* accum = empty + s.stages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.x * 128, split = blockIdx.y;
    const int kb_total = (s.K + 63) / 64;
    const int kb0 = split * s.kb_per_split;
    const int nkb = min(kb_total, kb0 + s.kb_per_split) - kb0;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
        for (int i = 0; i < s.stages; ++i) {
            tc::mbar_init(&full[i], 1);
            tc::mbar_init(&empty[i], 1);
        }
        tc::mbar_init(accum, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         tc::smem_u32(tmem_slot)),
                     "r"(s.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    pdl_trigger();
    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer: weights first (independent of the
        // previous kernel), then the activations after the PDL wait
        const int pre = min(nkb, s.stages);
        for (int kb = 0; kb < pre; ++kb) {
            tc::mbar_expect_tx(&full[kb], STAGE);
            tc::tma_load_2d(smem + kb * STAGE, &map_w, &full[kb], (kb0 + kb) * 64, n0);
        }
        pdl_wait();
        for (int kb = 0; kb < pre; ++kb)
            for (int g = 0; g < s.nbox; ++g)
                tc::tma_load_2d(smem + kb * STAGE + kWBytes + g * XB, &map_x, &full[kb], (kb0 + kb) * 64,
                                g * s.box_rows);
        int stage = pre % s.stages;
        uint32_t phase = pre == s.stages ? 1 : 0;
        for (int kb = pre; kb < nkb; ++kb) {
            tc::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = smem + stage * STAGE;
            tc::mbar_expect_tx(&full[stage], STAGE);
            const int kc = (kb0 + kb) * 64;
            tc::tma_load_2d(st, &map_w, &full[stage], kc, n0);
            for (int g = 0; g < s.nbox; ++g)
                tc::tma_load_2d(st + kWBytes + g * XB, &map_x, &full[stage], kc, g * s.box_rows);
            if (++stage == s.stages) {
                stage = 0;
                phase ^= 1;
            }
        }
    } else {
        pdl_wait();  // every global write of this kernel comes after this point
    }
    if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer (single thread)
        const uint32_t id = idesc(s.box_rows);
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = 0; kb < nkb; ++kb) {
            tc::mbar_wait(&full[stage], phase);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint8_t* st = smem + stage * STAGE;
            const uint64_t da = tc::smem_desc_sw128(st);
            for (int g = 0; g < s.nbox; ++g) {
                const uint64_t db = tc::smem_desc_sw128(st + kWBytes + g * XB);
#pragma unroll
                for (int k = 0; k < 4; ++k)  // +32 bytes per UMMA_K=16 inside the swizzle atom
                    tc::mma_bf16(tmem + g * 256, da + 2 * k, db + 2 * k, id, (kb | k) != 0);
            }
            tc::mma_commit(&empty[stage]);
            if (++stage == s.stages) {
                stage = 0;
                phase ^= 1;
            }
        }
        tc::mma_commit(accum);
    }
    __syncwarp();

    // ---------------- epilogue: thread = TMEM lane = weight row n
    tc::mbar_wait(accum, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int row = warp * 32 + lane;
    const int n = n0 + row;
    const bool nv = n < s.N;
    const uint32_t tl = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    for (int g = 0; g < s.nbox; ++g) {
        for (int c0 = 0; c0 < s.box_rows; c0 += 16) {
            const int m0 = g * s.box_rows + c0;
            if (m0 >= s.M) break;  // warp-uniform
            float v[16];
            tmem_ld16(tl + g * 256 + c0, v);
            if (s.mode == DEC_PARTIAL) {
                float* w = s.ws + (static_cast<size_t>(split) * s.M + m0) * s.N + n;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (nv && m0 + j < s.M) w[static_cast<size_t>(j) * s.N] = v[j];
            } else if (s.mode == DEC_SWIGLU) {
                __nv_bfloat16* y = static_cast<__nv_bfloat16*>(s.y) + n / 2;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float up = __shfl_xor_sync(0xffffffffu, v[j], 1);
                    if (!(lane & 1) && nv && m0 + j < s.M)
                        y[static_cast<size_t>(m0 + j) * s.ldy] = __float2bfloat16_rn(silu(v[j]) * up);
                }
            } else {
                const float b = (s.bias && nv) ? __ldg(s.bias + n) : 0.0f;
                __nv_bfloat16* y = static_cast<__nv_bfloat16*>(s.y) + n;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (nv && m0 + j < s.M)
                        y[static_cast<size_t>(m0 + j) * s.ldy] = __float2bfloat16_rn(v[j] + b);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "r"(s.tmem_cols));
}

}  // namespace dec
}  // namespace oppo
