// lmhead_dec.cuh — the actor's lm_head + in-block sampling for a decode batch
// (<= 128 tokens), swap-AB on tcgen05.
//
// One CTA per 256-id sampling block: the block's 256 vocabulary rows are the
// UMMA A operand (two M=128 MMAs per k16 step into two TMEM accumulators),
// the tokens are UMMA N.  Shared memory per stage holds 32 KB of weights and
// only the tokens that exist (the token-tiled kernel staged a 128-row,
// mostly zero-filled activation tile per block).  The epilogue keeps the
// token-tiled kernel's outputs and sampling rule (logits_tile): per token the
// block max, sum of exp, and the in-block inverse-CDF pick (first id whose
// running sum exceeds u * sum, ids in order, falling back to the block's last
// id), now with the 256 ids spread over the 128 TMEM lanes x 2 accumulators:
// warp-shuffle reductions and a warp scan, 16 tokens at a time.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "common.cuh"
#include "gemm.cuh"
#include "gemm_dec.cuh"

namespace oppo {
namespace lmh {

struct Shape {
    int M;           // tokens
    int Mp;          // tokens rounded to 16 (UMMA N, X box rows)
    int N;           // vocabulary
    int K;           // d_model
    int stages;
    int tmem_cols;   // pow2 >= 2 * Mp
    int n_tiles;     // sampling blocks per token row of `partials`
    float4* partials;        // [M][n_tiles]: max, sum-exp, pick (int bits), pick logit
    const uint64_t* keys;    // [M]
};

constexpr int kWBytes = 256 * 64 * 2;

static __global__ void __launch_bounds__(128, 1)
    lmhead_dec(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x, Shape s) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    const int XB = s.Mp * 128;
    const int STAGE = kWBytes + XB;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + s.stages * STAGE);
    uint64_t* empty = full + s.stages;
    uint64_t* accum = empty + s.stages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);
    float* red = reinterpret_cast<float*>(tmem_slot + 4);  // [4 warps][16 tokens] x 3

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.x, n0 = tile * 256;
    const int nkb = s.K / 64;
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
        const int pre = min(nkb, s.stages);
        for (int kb = 0; kb < pre; ++kb) {  // weights before the PDL wait
            tc::mbar_expect_tx(&full[kb], STAGE);
            tc::tma_load_2d(smem + kb * STAGE, &map_w, &full[kb], kb * 64, n0);
        }
        pdl_wait();
        for (int kb = 0; kb < pre; ++kb)
            tc::tma_load_2d(smem + kb * STAGE + kWBytes, &map_x, &full[kb], kb * 64, 0);
        int stage = pre % s.stages;
        uint32_t phase = pre == s.stages ? 1 : 0;
        for (int kb = pre; kb < nkb; ++kb) {
            tc::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = smem + stage * STAGE;
            tc::mbar_expect_tx(&full[stage], STAGE);
            tc::tma_load_2d(st, &map_w, &full[stage], kb * 64, n0);
            tc::tma_load_2d(st + kWBytes, &map_x, &full[stage], kb * 64, 0);
            if (++stage == s.stages) {
                stage = 0;
                phase ^= 1;
            }
        }
    } else {
        pdl_wait();
    }
    if (warp == 1 && lane == 0) {
        const uint32_t id = dec::idesc(s.Mp);
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = 0; kb < nkb; ++kb) {
            tc::mbar_wait(&full[stage], phase);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint8_t* st = smem + stage * STAGE;
            const uint64_t da0 = tc::smem_desc_sw128(st), da1 = tc::smem_desc_sw128(st + kWBytes / 2);
            const uint64_t db = tc::smem_desc_sw128(st + kWBytes);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                tc::mma_bf16(tmem, da0 + 2 * k, db + 2 * k, id, (kb | k) != 0);           // ids 0..127
                tc::mma_bf16(tmem + s.Mp, da1 + 2 * k, db + 2 * k, id, (kb | k) != 0);    // ids 128..255
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
    tc::mbar_wait(accum, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");

    // ---- epilogue: thread (warp w, lane l) holds ids i0 = 32w + l and i1 = 128 + i0
    const int nc = min(256, s.N - n0);
    const int i0 = warp * 32 + lane, i1 = 128 + i0;
    const bool v0ok = i0 < nc, v1ok = i1 < nc;
    const uint32_t tl = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    float* wmax = red;        // [4][16]
    float* wsum = red + 64;   // [4][16]
    float* wt0 = red + 128;   // [4][16] warp totals, ids 0..127
    float* wt1 = red + 192;   // [4][16] warp totals, ids 128..255
    int* wpick = reinterpret_cast<int*>(red + 256);  // [4][16] lowest crossing id per warp (or 1<<30)
    float* wlogit = red + 320;                        // [16] logit of the picked id
    for (int c0 = 0; c0 < s.Mp; c0 += 16) {
        if (c0 >= s.M) break;  // uniform
        float a[16], b[16];
        dec::tmem_ld16(tl + c0, a);
        dec::tmem_ld16(tl + s.Mp + c0, b);
        // 1. block max per token
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            float m = fmaxf(v0ok ? a[j] : -INFINITY, v1ok ? b[j] : -INFINITY);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) wmax[warp * 16 + j] = m;
        }
        __syncthreads();
        float mx[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
            mx[j] = fmaxf(fmaxf(wmax[j], wmax[16 + j]), fmaxf(wmax[32 + j], wmax[48 + j]));
        // 2. exp, block sum, and in-order inclusive prefix (warp scans)
        float e0[16], e1[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            e0[j] = v0ok ? __expf(a[j] - mx[j]) : 0.f;
            e1[j] = v1ok ? __expf(b[j] - mx[j]) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {  // inclusive warp scans
                const float p0 = __shfl_up_sync(0xffffffffu, e0[j], o);
                const float p1 = __shfl_up_sync(0xffffffffu, e1[j], o);
                if (lane >= o) {
                    e0[j] += p0;
                    e1[j] += p1;
                }
            }
            if (lane == 31) {
                wt0[warp * 16 + j] = e0[j];
                wt1[warp * 16 + j] = e1[j];
            }
        }
        __syncthreads();
        // 3. per token: block sum, this thread's global inclusive prefix, pick
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int m = c0 + j;
            float off0 = 0.f, tot0 = 0.f, off1 = 0.f, tot1 = 0.f;
#pragma unroll
            for (int w = 0; w < 4; ++w) {
                const float t0 = wt0[w * 16 + j], t1 = wt1[w * 16 + j];
                if (w < warp) {
                    off0 += t0;
                    off1 += t1;
                }
                tot0 += t0;
                tot1 += t1;
            }
            const float se = tot0 + tot1;
            const float thr = m < s.M ? key_uniform(s.keys[m] ^ kInBlockKey, static_cast<uint32_t>(tile)) * se : 0.f;
            const float p0 = off0 + e0[j], p1 = tot0 + off1 + e1[j];
            const unsigned c0m = __ballot_sync(0xffffffffu, v0ok && p0 > thr);
            const unsigned c1m = __ballot_sync(0xffffffffu, v1ok && p1 > thr);
            int cand = 1 << 30;
            if (c0m) cand = warp * 32 + __ffs(c0m) - 1;
            else if (c1m) cand = 128 + warp * 32 + __ffs(c1m) - 1;
            if (lane == 0) wpick[warp * 16 + j] = cand;
            if (lane == 0 && warp == 0) wsum[j] = se;
        }
        __syncthreads();
        // the picked id (first crossing, else the reference's fallback: the
        // block's last id); the thread holding it publishes its logit
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            int pick = min(min(wpick[j], wpick[16 + j]), min(wpick[32 + j], wpick[48 + j]));
            if (pick >= nc) pick = nc - 1;
            if (pick == i0) wlogit[j] = a[j];
            else if (pick == i1) wlogit[j] = b[j];
        }
        __syncthreads();
        if (threadIdx.x < 16 && c0 + static_cast<int>(threadIdx.x) < s.M) {
            const int j = threadIdx.x, m = c0 + j;
            int pick = min(min(wpick[j], wpick[16 + j]), min(wpick[32 + j], wpick[48 + j]));
            if (pick >= nc) pick = nc - 1;
            s.partials[static_cast<size_t>(m) * s.n_tiles + tile] =
                make_float4(mx[j], wsum[j], __int_as_float(n0 + pick), wlogit[j]);
        }
        __syncthreads();  // reductions of the next chunk reuse the scratch
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(s.tmem_cols));
}

}  // namespace lmh
}  // namespace oppo
