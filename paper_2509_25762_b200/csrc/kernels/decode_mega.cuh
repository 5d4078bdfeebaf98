// decode_mega.cuh — the actor's whole transformer stack for one decode
// iteration as ONE persistent kernel (bf16, <= 256 rows).
//
// A decode iteration at small batch is a chain of ~170 dependent, individually
// tiny launches; on B200 each launch boundary costs a few microseconds of
// drain + launch + dependency latency, which is what kept the iteration at
// ~8x the HBM floor.  Here one CTA per SM of the actor partition walks the
// 24 layers phase by phase, with a grid barrier (one global atomic + a
// generation flag) between phases:
//
//   norm1 -> qkv GEMM -> attention(+RoPE, KV append) -> O GEMM -> norm2
//         -> gate|up GEMM (+SwiGLU) -> down GEMM -> (next layer)
//
// GEMM phases are the swap-AB tcgen05 scheme of gemm_dec.cuh (128 weight rows
// on the TMEM lanes, tokens as UMMA N, TMA 128B-swizzled stages), work items =
// (weight tile, K split); split-K partials are folded by the consuming phase
// in split order (deterministic).  The TMEM accumulator is allocated once for
// the whole kernel; the TMA/MMA pipeline state persists across items and
// phases, and at the end of every phase the producer thread already issues
// the WEIGHT loads of its first item of the next GEMM phase (weights never
// depend on the barrier), so weight streaming overlaps the barrier and the
// non-GEMM phases.  Attention work items are (row, KV head, split); splits
// of a row merge through a workspace, the last-arriving split does the merge.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>

#include "attn_dec.cuh"
#include "attn_mma.cuh"
#include "common.cuh"
#include "gemm.cuh"
#include "gemm_dec.cuh"
#include "model.cuh"

namespace oppo {
namespace mega {

struct LayerP {
    CUtensorMap w[4];  // qkv, o, gate|up, down: [N, K] bf16, box 128 rows x 64
    const float* bqkv;
    const float* ln1;
    const float* ln2;
    const void* pad;
};

enum { W_QKV = 0, W_O = 1, W_GU = 2, W_DN = 3 };

struct Args {
    int M, Mp, D, H, KV, HD, F, L;
    int qkvw, qw;
    float* x;              // residual [M, D] fp32
    __nv_bfloat16* h;      // normed rows [M, D]
    __nv_bfloat16* attn;   // attention out [M, qw]
    __nv_bfloat16* ff;     // SwiGLU out [M, F]
    float* ws;             // split-K partials [split][M][N]
    float* aws;            // attention split partials [M*KV][att_sp][SLOT]
    int* acnt;             // attention merge counters [M*KV] (zero on entry and exit)
    unsigned* bar;         // grid barrier {count, generation}
    const LayerP* layers;  // [L] (device)
    KvView kv;
    const int32_t* slot;
    const int32_t* pos;
    int sp[4], kbps[4];    // per GEMM: K splits (= ceil(k blocks / kbps)) and k blocks per split
    int att_sp;            // attention splits per (row, KV head)
    int stages, stage_bytes, attn_off, tmem_cols;
    int first_np;          // split-K partials pending in ws from before the kernel
    float eps, theta;
    unsigned long long* trace;  // optional: %globaltimer after every barrier (CTA 0)
    int barriers_only;          // perf diagnosis: skip all phase work (results garbage)
    int bar_ra;                 // 1: release/acquire barrier (grid_sync_ra)
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

// --------------------------------------------------------------- barrier
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void grid_sync(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> later TMA reads
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(32);
        }
        __threadfence();
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    __syncthreads();
}

// Same barrier with release/acquire atomics instead of full fences: the
// arrival is an atom.add.release.gpu (orders this CTA's prior writes), the
// wait an ld.acquire.gpu poll of the generation word.
__device__ __forceinline__ void grid_sync_ra(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g, old;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        if (old == gridDim.x - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(bar) : "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar + 1) : "memory");
        } else {
            unsigned cur;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
            } while (cur == g);
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> later TMA reads
    }
    __syncthreads();
}

__device__ __forceinline__ void sync_all(const Args& a) {
    if (a.bar_ra) grid_sync_ra(a.bar);
    else grid_sync(a.bar);
}

// ------------------------------------------------------------ GEMM phase
struct Pipe {
    int stage = 0;        // producer and MMA walk the stages in the same order
    uint32_t phase = 0;
    int mstage = 0;
    uint32_t mphase = 0;
    uint32_t acc_parity = 0;
    uint32_t free_parity = 0;
    bool first_item = true;
    int pre = 0;          // producer: stages holding prefetched W of the next item
    int pre_item = -1;    // which item (of which GEMM) they belong to
    int pre_gemm = -1;
};

struct Smem {
    uint8_t* stages;
    uint64_t* full;
    uint64_t* empty;
    uint64_t* accum;
    uint64_t* tfree;
    uint32_t* tmem_slot;
    float* red;
    uint8_t* attn;
};

__device__ __forceinline__ int gemm_n(const Args& a, int g) {
    return g == W_QKV ? a.qkvw : g == W_O ? a.D : g == W_GU ? 2 * a.F : a.D;
}
__device__ __forceinline__ int gemm_k(const Args& a, int g) {
    return g == W_QKV ? a.D : g == W_O ? a.qw : g == W_GU ? a.D : a.F;
}
__device__ __forceinline__ int gemm_items(const Args& a, int g) {
    return ((gemm_n(a, g) + 127) / 128) * a.sp[g];
}
__device__ __forceinline__ void item_range(const Args& a, int g, int item, int& tile, int& k0, int& nkb) {
    const int tiles = (gemm_n(a, g) + 127) / 128;
    tile = item % tiles;
    const int split = item / tiles;
    const int kbt = gemm_k(a, g) / 64;
    k0 = split * a.kbps[g];
    nkb = max(0, min(kbt, k0 + a.kbps[g]) - k0);
}

// producer only: issue the weight loads of (gemm g, item) into the next
// free stages, up to the pipeline depth (arms each stage for W + X bytes)
__device__ __forceinline__ void prefetch_w(const Args& a, const Smem& sm, Pipe& p, int layer, int g,
                                           int item) {
    p.pre = 0;
    p.pre_item = -1;
    if (layer >= a.L || item >= gemm_items(a, g)) return;
    int tile, k0, nkb;
    item_range(a, g, item, tile, k0, nkb);
    const CUtensorMap* wm = &a.layers[layer].w[g];
    const int n = min(nkb, a.stages);
    for (int kb = 0; kb < n; ++kb) {
        tc::mbar_wait(&sm.empty[p.stage], p.phase ^ 1);
        tc::mbar_expect_tx(&sm.full[p.stage], a.stage_bytes);
        tc::tma_load_2d(sm.stages + p.stage * a.stage_bytes, wm, &sm.full[p.stage], (k0 + kb) * 64, tile * 128);
        if (++p.stage == a.stages) {
            p.stage = 0;
            p.phase ^= 1;
        }
    }
    p.pre = n;
    p.pre_item = item;
    p.pre_gemm = g;
}

// One GEMM phase: every item of this CTA.  X = activation map (rows = M).
// PARTIAL -> ws[split][m][n]; SWIGLU -> ff.
static __device__ void gemm_phase(const Args& a, const Smem& sm, Pipe& p, uint32_t tmem, int layer, int g,
                           const CUtensorMap* xmap, int mode, int next_layer, int next_g) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int N = gemm_n(a, g), tiles = (N + 127) / 128;
    const int items = gemm_items(a, g);
    const CUtensorMap* wm = &a.layers[layer].w[g];
    const uint32_t idesc = dec::idesc(a.Mp);
    const int xb = dec::kWBytes;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        int tile, k0, nkb;
        item_range(a, g, item, tile, k0, nkb);
        const int split = item / tiles;
        if (warp == 0 && lane == 0) {
            // stages [stage - pre, stage) already hold this item's W (prefetched)
            int pre = (p.pre_item == item && p.pre_gemm == g) ? p.pre : 0;
            int st = p.stage - pre;
            uint32_t ph = p.phase;
            if (st < 0) {
                st += a.stages;
                ph ^= 1;
            }
            for (int kb = 0; kb < pre; ++kb) {  // X of the prefetched stages
                tc::tma_load_2d(sm.stages + st * a.stage_bytes + xb, xmap, &sm.full[st], (k0 + kb) * 64, 0);
                if (++st == a.stages) st = 0;
            }
            for (int kb = pre; kb < nkb; ++kb) {
                tc::mbar_wait(&sm.empty[p.stage], p.phase ^ 1);
                uint8_t* sb = sm.stages + p.stage * a.stage_bytes;
                tc::mbar_expect_tx(&sm.full[p.stage], a.stage_bytes);
                tc::tma_load_2d(sb, wm, &sm.full[p.stage], (k0 + kb) * 64, tile * 128);
                tc::tma_load_2d(sb + xb, xmap, &sm.full[p.stage], (k0 + kb) * 64, 0);
                if (++p.stage == a.stages) {
                    p.stage = 0;
                    p.phase ^= 1;
                }
            }
            p.pre = 0;
            p.pre_item = -1;
        }
        if (warp == 1 && lane == 0) {
            if (!p.first_item) {  // the previous item's epilogue has read TMEM
                tc::mbar_wait(sm.tfree, p.free_parity);
                p.free_parity ^= 1;
            }
            p.first_item = false;
            for (int kb = 0; kb < nkb; ++kb) {
                tc::mbar_wait(&sm.full[p.mstage], p.mphase);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint8_t* sb = sm.stages + p.mstage * a.stage_bytes;
                const uint64_t da = tc::smem_desc_sw128(sb), db = tc::smem_desc_sw128(sb + xb);
#pragma unroll
                for (int k = 0; k < 4; ++k) tc::mma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
                tc::mma_commit(&sm.empty[p.mstage]);
                if (++p.mstage == a.stages) {
                    p.mstage = 0;
                    p.mphase ^= 1;
                }
            }
            tc::mma_commit(sm.accum);
        }
        __syncwarp();
        // ---- epilogue: thread = weight row n of this tile
        tc::mbar_wait(sm.accum, p.acc_parity);
        p.acc_parity ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;");
        const int n = tile * 128 + warp * 32 + lane;
        const bool nv = n < N && nkb > 0;
        const uint32_t tl = tmem + (static_cast<uint32_t>(warp * 32) << 16);
        for (int c0 = 0; c0 < a.Mp; c0 += 16) {
            if (c0 >= a.M) break;
            float v[16];
            dec::tmem_ld16(tl + c0, v);
            if (mode == DEC_PARTIAL) {
                float* w = a.ws + (static_cast<size_t>(split) * a.M + c0) * N + n;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < a.M && n < N) w[static_cast<size_t>(j) * N] = nv ? v[j] : 0.f;
            } else {
                __nv_bfloat16* y = a.ff + n / 2;
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float up = __shfl_xor_sync(0xffffffffu, v[j], 1);
                    if (!(lane & 1) && n < N && c0 + j < a.M)
                        y[static_cast<size_t>(c0 + j) * a.F] = __float2bfloat16_rn(silu(v[j]) * up);
                }
            }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        mbar_arrive(sm.tfree);  // 128 arrivals free the accumulator
    }
    // weights of this CTA's first item of the next GEMM phase, ahead of the barrier
    if (warp == 0 && lane == 0 && next_g >= 0) prefetch_w(a, sm, p, next_layer, next_g, blockIdx.x);
}

// ------------------------------------------------------------ norm phase
// x[r] += sum_s part[s][r] (split order); h[r] = x[r] * rsqrt(mean x^2 + eps) * g
static __device__ void norm_phase(const Args& a, const Smem& sm, const float* gamma, int np, int pstride_n) {
    const int tid = threadIdx.x, nv = a.D >> 2;
    constexpr int kCols = 7;  // 128 threads x 7 float4 >= 3584
    for (int r = blockIdx.x; r < a.M; r += gridDim.x) {
        float4* xr = reinterpret_cast<float4*>(a.x + static_cast<size_t>(r) * a.D);
        float4 v[kCols];
        float ss = 0.f;
        const size_t ps = static_cast<size_t>(a.M) * pstride_n / 4;
#pragma unroll
        for (int i = 0; i < kCols; ++i) {
            const int c = tid + 128 * i;
            if (c >= nv) continue;
            float4 acc = xr[c];
            const float4* pc = reinterpret_cast<const float4*>(a.ws) + static_cast<size_t>(r) * nv + c;
            for (int s0 = 0; s0 < np; s0 += 8) {  // 8 split loads in flight, summed in split order
                float4 pv[8];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    pv[k] = s0 + k < np ? __ldcg(pc + (s0 + k) * ps) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (s0 + k >= np) break;
                    acc.x += pv[k].x; acc.y += pv[k].y; acc.z += pv[k].z; acc.w += pv[k].w;
                }
            }
            if (np > 0) xr[c] = acc;
            v[i] = acc;
            ss += acc.x * acc.x + acc.y * acc.y + acc.z * acc.z + acc.w * acc.w;
        }
        ss = warp_sum(ss);
        if ((tid & 31) == 0) sm.red[tid >> 5] = ss;
        __syncthreads();
        ss = sm.red[0] + sm.red[1] + sm.red[2] + sm.red[3];
        __syncthreads();
        const float inv = rsqrtf(ss / a.D + a.eps);
        __nv_bfloat16* orow = a.h + static_cast<size_t>(r) * a.D;
#pragma unroll
        for (int i = 0; i < kCols; ++i) {
            const int c = tid + 128 * i;
            if (c >= nv) continue;
            const float4 g = reinterpret_cast<const float4*>(gamma)[c];
            orow[4 * c] = __float2bfloat16_rn(v[i].x * inv * g.x);
            orow[4 * c + 1] = __float2bfloat16_rn(v[i].y * inv * g.y);
            orow[4 * c + 2] = __float2bfloat16_rn(v[i].z * inv * g.z);
            orow[4 * c + 3] = __float2bfloat16_rn(v[i].w * inv * g.w);
        }
    }
}

// -------------------------------------------------------- attention phase
// item = (row, KV head, split): attn_dec's phases 1-3 on this CTA, then the
// split partials merge through a.aws; the last-arriving split merges.
template <int HD>
__device__ void attn_phase(const Args& a, const Smem& sm, int layer, int np_qkv) {
    using namespace am;
    using Cf = AttnDecCfg<HD>;
    constexpr int TP = Cf::TP, LDS = Cf::LDS, NT = TP / 8, DT = HD / 8;
    const int KV = a.KV, H = a.H, G = H / KV, nsp = a.att_sp;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    uint8_t* kvbuf = sm.attn;
    auto sQ = reinterpret_cast<__nv_bfloat16(*)[LDS]>(kvbuf + 4 * Cf::WARP_BYTES);
    float* fq = reinterpret_cast<float*>(kvbuf);
    const float* bias = a.layers[layer].bqkv;
    const int items = a.M * KV * nsp;
    const int width = a.qkvw;
    const size_t pstride = static_cast<size_t>(a.M) * width;
    __shared__ int s_last;
    for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int z = item % nsp, rh = item / nsp, r = rh / KV, h = rh % KV;
        const int slot = a.slot[r], pos = a.pos[r], ctx = pos + 1;
        const int slen = (ctx + nsp - 1) / nsp;
        const int p_begin = min(ctx, z * slen), p_end = min(ctx, p_begin + slen);
        const bool owner = pos >= p_begin && pos < p_end;
        for (int i = tid; i < (G + 2) * HD; i += 128) {
            const int gi = i / HD, d = i % HD;
            const int col = gi < G ? (h * G + gi) * HD + d : gi == G ? (H + h) * HD + d : (H + KV + h) * HD + d;
            const float* pp = a.ws + static_cast<size_t>(r) * width + col;
            float acc = 0.f;
            for (int s0 = 0; s0 < np_qkv; s0 += 8) {  // 8 split loads in flight, split order
                float pv[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) pv[k] = s0 + k < np_qkv ? __ldcg(pp + (s0 + k) * pstride) : 0.f;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (s0 + k >= np_qkv) break;
                    acc += pv[k];
                }
            }
            fq[gi * HD + d] = tof(fromf<__nv_bfloat16>(acc + bias[col]));
        }
        __syncthreads();
        const int half = HD / 2;
        for (int i = tid; i < (G + 1) * half; i += 128) {
            const int gi = i / half, d = i % half;
            const float inv_freq = __powf(a.theta, -2.0f * d / HD);
            float sn, cs;
            sincosf(pos * inv_freq, &sn, &cs);
            const float x1 = fq[gi * HD + d], x2 = fq[gi * HD + d + half];
            const float y1 = x1 * cs - x2 * sn, y2 = x2 * cs + x1 * sn;
            if (gi < G) {
                sQ[gi][d] = fromf<__nv_bfloat16>(y1);
                sQ[gi][d + half] = fromf<__nv_bfloat16>(y2);
            } else if (owner) {
                __nv_bfloat16* kc = static_cast<__nv_bfloat16*>(a.kv.k) + kv_index<__nv_bfloat16>(a.kv, layer, slot, pos, h);
                kc[d] = fromf<__nv_bfloat16>(y1);
                kc[d + half] = fromf<__nv_bfloat16>(y2);
            }
        }
        if (owner) {
            __nv_bfloat16* vc = static_cast<__nv_bfloat16*>(a.kv.v) + kv_index<__nv_bfloat16>(a.kv, layer, slot, pos, h);
            for (int d = tid; d < HD; d += 128) vc[d] = fromf<__nv_bfloat16>(fq[(G + 1) * HD + d]);
        }
        for (int i = tid; i < (16 - G) * HD; i += 128) sQ[G + i / HD][i % HD] = fromf<__nv_bfloat16>(0.f);
        __threadfence_block();
        __syncthreads();
        const int gid = lane >> 2, tig = lane & 3;
        const int row0 = gid, row1 = gid + 8;
        const bool ok0 = row0 < G, ok1 = row1 < G;
        uint32_t qf[HD / 16][4];
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
            const int c = kk * 16 + tig * 2;
            qf[kk][0] = *reinterpret_cast<const uint32_t*>(&sQ[row0][c]);
            qf[kk][1] = *reinterpret_cast<const uint32_t*>(&sQ[row1][c]);
            qf[kk][2] = *reinterpret_cast<const uint32_t*>(&sQ[row0][c + 8]);
            qf[kk][3] = *reinterpret_cast<const uint32_t*>(&sQ[row1][c + 8]);
        }
        auto sK = reinterpret_cast<__nv_bfloat16(*)[TP][LDS]>(kvbuf + warp * Cf::WARP_BYTES);
        auto sV = reinterpret_cast<__nv_bfloat16(*)[TP][LDS]>(kvbuf + warp * Cf::WARP_BYTES + 2 * TP * LDS * 2);
        const float scale = rsqrtf(static_cast<float>(HD)) * 1.4426950408889634f;
        float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
        float o[DT][4];
#pragma unroll
        for (int d = 0; d < DT; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.f;
        const __nv_bfloat16* kc = static_cast<const __nv_bfloat16*>(a.kv.k);
        const __nv_bfloat16* vc = static_cast<const __nv_bfloat16*>(a.kv.v);
        auto load_tile = [&](int buf, int t0) {
            constexpr int CHUNKS = TP * HD / 8;
#pragma unroll
            for (int c = lane; c < CHUNKS; c += 32) {
                const int pp = c / (HD / 8), e = (c % (HD / 8)) * 8;
                const int ps = t0 + pp;
                const bool valid = ps < p_end;
                const size_t base = valid ? kv_index<__nv_bfloat16>(a.kv, layer, slot, ps, h) + e : 0;
                cp_async16(&sK[buf][pp][e], kc + base, valid);
                cp_async16(&sV[buf][pp][e], vc + base, valid);
            }
            cp_async_commit();
        };
        int buf = 0;
        const int first = p_begin + warp * TP;
        if (first < p_end) load_tile(0, first);
        for (int t0 = first; t0 < p_end; t0 += 4 * TP) {
            if (t0 + 4 * TP < p_end) {
                load_tile(buf ^ 1, t0 + 4 * TP);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncwarp();
            float s[NT][4];
#pragma unroll
            for (int j = 0; j < NT; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
                for (int j = 0; j < NT; j += 2) {
                    const int mi = lane >> 3, rr = lane & 7;
                    uint32_t b[4];
                    ldsm_x4(b, &sK[buf][(j + (mi >> 1)) * 8 + rr][kk * 16 + (mi & 1) * 8]);
                    mma16816(s[j], qf[kk], b[0], b[1]);
                    mma16816(s[j + 1], qf[kk], b[2], b[3]);
                }
            }
            float mx0 = m0, mx1 = m1;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int ps = t0 + j * 8 + tig * 2 + (c & 1);
                    const bool ok = ps < p_end && (c >= 2 ? ok1 : ok0);
                    s[j][c] = ok ? s[j][c] * scale : -INFINITY;
                }
                mx0 = fmaxf(mx0, fmaxf(s[j][0], s[j][1]));
                mx1 = fmaxf(mx1, fmaxf(s[j][2], s[j][3]));
            }
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
            mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
            mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
            const float c0 = mx0 == -INFINITY ? 1.f : exp2f(m0 - mx0);
            const float c1 = mx1 == -INFINITY ? 1.f : exp2f(m1 - mx1);
            m0 = mx0;
            m1 = mx1;
            l0 *= c0;
            l1 *= c1;
#pragma unroll
            for (int d = 0; d < DT; ++d) {
                o[d][0] *= c0;
                o[d][1] *= c0;
                o[d][2] *= c1;
                o[d][3] *= c1;
            }
            uint32_t pa[NT / 2][4];
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const float e0 = m0 == -INFINITY ? 0.f : exp2f(s[j][0] - m0);
                const float e1 = m0 == -INFINITY ? 0.f : exp2f(s[j][1] - m0);
                const float e2 = m1 == -INFINITY ? 0.f : exp2f(s[j][2] - m1);
                const float e3 = m1 == -INFINITY ? 0.f : exp2f(s[j][3] - m1);
                l0 += e0 + e1;
                l1 += e2 + e3;
                pa[j >> 1][(j & 1) * 2 + 0] = pack_bf16(e0, e1);
                pa[j >> 1][(j & 1) * 2 + 1] = pack_bf16(e2, e3);
            }
#pragma unroll
            for (int kk = 0; kk < NT / 2; ++kk) {
#pragma unroll
                for (int d = 0; d < DT; d += 2) {
                    const int mi = lane >> 3, rr = lane & 7;
                    uint32_t b[4];
                    ldsm_x4_t(b, &sV[buf][kk * 16 + (mi & 1) * 8 + rr][(d + (mi >> 1)) * 8]);
                    mma16816(o[d], pa[kk], b[0], b[1]);
                    mma16816(o[d + 1], pa[kk], b[2], b[3]);
                }
            }
            __syncwarp();
            buf ^= 1;
        }
        l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
        l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
        __syncthreads();  // every warp is done with its K/V buffers
        // warp partials -> local slots 0..3; merge them into one CTA partial
        float* loc = reinterpret_cast<float*>(kvbuf) + warp * Cf::SLOT;
#pragma unroll
        for (int d = 0; d < DT; ++d) {
            const int c = d * 8 + tig * 2;
            *reinterpret_cast<float2*>(loc + row0 * HD + c) = make_float2(o[d][0], o[d][1]);
            *reinterpret_cast<float2*>(loc + row1 * HD + c) = make_float2(o[d][2], o[d][3]);
        }
        if (tig == 0) {
            *reinterpret_cast<float2*>(loc + 16 * HD + row0 * 2) = make_float2(m0, l0);
            *reinterpret_cast<float2*>(loc + 16 * HD + row1 * 2) = make_float2(m1, l1);
        }
        __syncthreads();
        const float* lb = reinterpret_cast<const float*>(kvbuf);
        float* part = a.aws + (static_cast<size_t>(rh) * nsp + z) * Cf::SLOT;
        // CTA partial (natural: unnormalised O and (max, sum) in the exp2 domain)
        for (int e = tid; e < G * HD; e += 128) {
            const int g = e / HD;
            float mx = -INFINITY;
            for (int w = 0; w < 4; ++w) mx = fmaxf(mx, lb[w * Cf::SLOT + 16 * HD + g * 2]);
            float L = 0.f, O = 0.f;
            for (int w = 0; w < 4; ++w) {
                const float ms = lb[w * Cf::SLOT + 16 * HD + g * 2];
                const float wgt = ms == -INFINITY ? 0.f : exp2f(ms - mx);
                L += lb[w * Cf::SLOT + 16 * HD + g * 2 + 1] * wgt;
                O += lb[w * Cf::SLOT + e] * wgt;
            }
            if (nsp == 1) {
                a.attn[(static_cast<size_t>(r) * H + h * G + g) * HD + (e % HD)] =
                    __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
            } else {
                part[e] = O;
                if (e % HD == 0) {
                    part[16 * HD + g * 2] = mx;
                    part[16 * HD + g * 2 + 1] = L;
                }
            }
        }
        if (nsp > 1) {
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                const int prev = atomicAdd(&a.acnt[rh], 1);
                s_last = prev == nsp - 1;
                if (s_last) a.acnt[rh] = 0;
            }
            __syncthreads();
            if (s_last) {
                __threadfence();
                const float* pb = a.aws + static_cast<size_t>(rh) * nsp * Cf::SLOT;
                for (int e = tid; e < G * HD; e += 128) {
                    const int g = e / HD;
                    float mx = -INFINITY;
                    for (int s = 0; s < nsp; ++s) mx = fmaxf(mx, __ldcg(pb + s * Cf::SLOT + 16 * HD + g * 2));
                    float L = 0.f, O = 0.f;
                    for (int s = 0; s < nsp; ++s) {
                        const float ms = __ldcg(pb + s * Cf::SLOT + 16 * HD + g * 2);
                        const float wgt = ms == -INFINITY ? 0.f : exp2f(ms - mx);
                        L += __ldcg(pb + s * Cf::SLOT + 16 * HD + g * 2 + 1) * wgt;
                        O += __ldcg(pb + s * Cf::SLOT + e) * wgt;
                    }
                    a.attn[(static_cast<size_t>(r) * H + h * G + g) * HD + (e % HD)] =
                        __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
                }
            }
        }
        __syncthreads();  // smem reused by the next item
    }
}

// ---------------------------------------------------------------- kernel
template <int HD>
__global__ void __launch_bounds__(128, 1)
    decode_layers(const __grid_constant__ CUtensorMap xm_h, const __grid_constant__ CUtensorMap xm_attn,
                  const __grid_constant__ CUtensorMap xm_ff, const __grid_constant__ Args a) {
    extern __shared__ uint8_t msm_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(msm_raw) + 1023) & ~uintptr_t(1023));
    Smem sm;
    sm.stages = base;
    sm.attn = base + a.attn_off;
    uint8_t* tail = sm.attn + AttnDecCfg<HD>::SMEM;
    sm.full = reinterpret_cast<uint64_t*>(tail);
    sm.empty = sm.full + a.stages;
    sm.accum = sm.empty + a.stages;
    sm.tfree = sm.accum + 1;
    sm.tmem_slot = reinterpret_cast<uint32_t*>(sm.tfree + 1);
    sm.red = reinterpret_cast<float*>(sm.tmem_slot + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < a.stages; ++i) {
            tc::mbar_init(&sm.full[i], 1);
            tc::mbar_init(&sm.empty[i], 1);
        }
        tc::mbar_init(sm.accum, 1);
        tc::mbar_init(sm.tfree, 128);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xm_h)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xm_attn)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&xm_ff)) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         tc::smem_u32(sm.tmem_slot)),
                     "r"(a.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *sm.tmem_slot;
    Pipe p;
    if (warp == 0 && lane == 0) prefetch_w(a, sm, p, 0, W_QKV, blockIdx.x);  // before the PDL wait
    pdl_wait();
    int np = a.first_np;
    int tix = 1;
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[0] = gtimer();
    if (a.barriers_only) {
        int tix = 1;
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[0] = gtimer();
        for (int k = 0; k < 7 * a.L; ++k) {
            sync_all(a);
            if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[tix++] = gtimer();
        }
        np = 0;
    }
    for (int l = 0; l < (a.barriers_only ? 0 : a.L); ++l) {
        const LayerP& L = a.layers[l];
        norm_phase(a, sm, L.ln1, np, a.D);
        sync_all(a);
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[tix++] = gtimer();
        gemm_phase(a, sm, p, tmem, l, W_QKV, &xm_h, DEC_PARTIAL, l, W_O);
        sync_all(a);
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[tix++] = gtimer();
        attn_phase<HD>(a, sm, l, a.sp[W_QKV]);
        sync_all(a);
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[tix++] = gtimer();
        gemm_phase(a, sm, p, tmem, l, W_O, &xm_attn, DEC_PARTIAL, l, W_GU);
        sync_all(a);
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[tix++] = gtimer();
        norm_phase(a, sm, L.ln2, a.sp[W_O], a.D);
        sync_all(a);
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[tix++] = gtimer();
        gemm_phase(a, sm, p, tmem, l, W_GU, &xm_h, DEC_SWIGLU, l, W_DN);
        sync_all(a);
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[tix++] = gtimer();
        gemm_phase(a, sm, p, tmem, l, W_DN, &xm_ff, DEC_PARTIAL, l + 1, W_QKV);
        np = a.sp[W_DN];
        sync_all(a);
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) a.trace[tix++] = gtimer();
    }
    pdl_trigger();
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
}

}  // namespace mega
}  // namespace oppo
