// attn_train_mma.cuh — causal GQA attention of the full-parameter update on
// the tensor cores (mma.sync m16n8k16 bf16, fp32 accumulation), FA2 style:
//   fwd: one CTA per (64-query block, q head), 4 warps x 16 query rows,
//        online softmax over the causal key blocks; writes O and the
//        per-(row, head) log-sum-exp;
//   dq:  one CTA per (64-query block, q head): P and dS recomputed per key
//        block, dQ += dS K;
//   dkv: one CTA per (64-key block, kv head), 4 warps x 16 keys: loops over
//        the G query heads of the group and the query blocks at or after the
//        key block; dV += P^T dO, dK += dS^T Q.
// Rows of a sequence are contiguous in the training layout; a block never
// straddles two sequences (TBlk: sequence start, length, block start).
// Semantics as the SIMT kernels in train.cuh (which the fp32 engine uses and
// the tests compare against); the S = QK^T, P.V, dP = dO V^T, dS K, ... tiles
// are the GEMM-shaped part of attention, so they go to the tensor cores.
#pragma once

#include "common.cuh"
#include "train.cuh"

namespace oppo {
namespace train {

constexpr int kMBlk = 64;  // rows per block of the mma kernels

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint32_t ld32(const __nv_bfloat16* p) { return *reinterpret_cast<const uint32_t*>(p); }

// Transpose of the forward's rotate-half RoPE (the backward of q / k) applied
// to a thread's accumulator fragment of one row: dims dt*8 + 2*tq + e and
// their rotation partners dims + HD/2 (dt + HD/16) sit in the same thread.
// Same angle arithmetic as train::rope_rows (powf, sincosf) at position pos.
template <int HD>
__device__ __forceinline__ void rope_bwd_frag(float (&f)[HD / 8][4], int i, int tq, int pos, float theta) {
#pragma unroll
    for (int dt = 0; dt < HD / 16; ++dt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int d = dt * 8 + 2 * tq + e;
            float sn, cs;
            sincosf(static_cast<float>(pos) * powf(theta, -2.0f * d / HD), &sn, &cs);
            const float a = f[dt][2 * i + e], b = f[dt + HD / 16][2 * i + e];
            f[dt][2 * i + e] = a * cs + b * sn;
            f[dt + HD / 16][2 * i + e] = b * cs - a * sn;
        }
}

template <int HD>
struct MmaT {
    static constexpr int RS = HD + 8;        // row-major tile stride (elements)
    static constexpr int ROW = kMBlk * RS;   // elements of a row-major tile
    static constexpr int SMEM_FWD = 5 * ROW * 2;  // Q + double-buffered K, V
    static constexpr int SMEM_DQ = 6 * ROW * 2;   // Q, dO + double-buffered K, V
    static constexpr int SMEM_DKV = 6 * ROW * 2 + 4 * kMBlk * 4;  // K, V + double-buffered Q, dO, lse, dvec
};

// rows [r0, r0 + n) of columns [col, col + HD) of a row-major bf16 matrix ->
// smem (row-major, stride RS; zero rows beyond n)
template <int HD>
__device__ __forceinline__ void load_rows(__nv_bfloat16* dst, const __nv_bfloat16* __restrict__ src, size_t ld,
                                          int r0, int n, int col) {
    using M = MmaT<HD>;
    constexpr int VPR = HD / 8;  // 16-byte vectors per row
    for (int i = threadIdx.x; i < kMBlk * VPR; i += blockDim.x) {
        const int r = i / VPR, c = (i % VPR) * 8;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r < n) v = *reinterpret_cast<const uint4*>(src + static_cast<size_t>(r0 + r) * ld + col + c);
        *reinterpret_cast<uint4*>(dst + r * M::RS + c) = v;
    }
}

// The same with cp.async (16-byte copies into smem, L2 only); rows beyond n
// are zeroed with plain stores.  Complete after cp_async_wait + __syncthreads.
template <int HD>
__device__ __forceinline__ void load_rows_async(__nv_bfloat16* dst, const __nv_bfloat16* __restrict__ src, size_t ld,
                                                int r0, int n, int col) {
    using M = MmaT<HD>;
    constexpr int VPR = HD / 8;
    for (int i = threadIdx.x; i < kMBlk * VPR; i += blockDim.x) {
        const int r = i / VPR, c = (i % VPR) * 8;
        __nv_bfloat16* d = dst + r * M::RS + c;
        if (r < n) {
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(d))),
                         "l"(src + static_cast<size_t>(r0 + r) * ld + col + c)
                         : "memory");
        } else {
            *reinterpret_cast<uint4*>(d) = make_uint4(0, 0, 0, 0);
        }
    }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// A fragment (16 rows x 16 k) of a row-major smem tile at (row0, k0)
template <int HD>
__device__ __forceinline__ void frag_a(uint32_t (&a)[4], const __nv_bfloat16* t, int row0, int k0, int g, int tq) {
    using M = MmaT<HD>;
    a[0] = ld32(t + (row0 + g) * M::RS + k0 + 2 * tq);
    a[1] = ld32(t + (row0 + g + 8) * M::RS + k0 + 2 * tq);
    a[2] = ld32(t + (row0 + g) * M::RS + k0 + 2 * tq + 8);
    a[3] = ld32(t + (row0 + g + 8) * M::RS + k0 + 2 * tq + 8);
}

// acc[nt] (16 x 64, nt = 8-column tiles) = A(16 rows of `a` tile) . B^T where
// B's rows are the 64 rows of `b` tile (both row-major over HD)
template <int HD>
__device__ __forceinline__ void qk_tile(float (&acc)[8][4], const __nv_bfloat16* a, int arow0,
                                        const __nv_bfloat16* b, int g, int tq) {
    using M = MmaT<HD>;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[nt][c] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD; kk += 16) {
        uint32_t af[4];
        frag_a<HD>(af, a, arow0, kk, g, tq);
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
            const __nv_bfloat16* br = b + (nt * 8 + g) * M::RS + kk + 2 * tq;
            mma16816(acc[nt], af, ld32(br), ld32(br + 8));
        }
    }
}

// out[dt] (16 x HD) += P (16 x 64 in registers, C layout) . B where B is a
// row-major smem tile [64 keys][HD] (stride RS): the col-major B fragments
// (pairs along the key dimension) come straight from ldmatrix .trans, two
// 8-column d blocks per ldmatrix.x4 -- no transposed copy of the tile.
__device__ __forceinline__ void ldsm_x4_trans(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
}
template <int HD>
__device__ __forceinline__ void pv_tile(float (&out)[HD / 8][4], const float (&p)[8][4], const __nv_bfloat16* b,
                                        int lane) {
    using M = MmaT<HD>;
    // this lane's ldmatrix row: matrix lane/8 = (key half, d block), row lane%8
    const int key_off = (lane & 7) + ((lane >> 3) & 1) * 8, d_off = (lane >> 4) * 8;
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {
        uint32_t a[4];
        a[0] = pack_bf16(p[2 * kc][0], p[2 * kc][1]);
        a[1] = pack_bf16(p[2 * kc][2], p[2 * kc][3]);
        a[2] = pack_bf16(p[2 * kc + 1][0], p[2 * kc + 1][1]);
        a[3] = pack_bf16(p[2 * kc + 1][2], p[2 * kc + 1][3]);
#pragma unroll
        for (int dt = 0; dt < HD / 8; dt += 2) {
            uint32_t r[4];
            ldsm_x4_trans(r, b + (kc * 16 + key_off) * M::RS + dt * 8 + d_off);
            mma16816(out[dt], a, r[0], r[1]);
            mma16816(out[dt + 1], a, r[2], r[3]);
        }
    }
}

template <int HD>
__global__ void __launch_bounds__(128) attn_fwd_mma(const TBlk* __restrict__ blks, const __nv_bfloat16* __restrict__ qkv,
                                                    int ld, int H, int KV, __nv_bfloat16* __restrict__ out,
                                                    float* __restrict__ lse) {
    using M = MmaT<HD>;
    extern __shared__ __align__(16) uint8_t smraw[];
    __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(smraw);
    const TBlk b = blks[blockIdx.x];
    const int h = blockIdx.y, kvh = h / (H / KV);
    const int nq = min(kMBlk, b.len - b.q0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
    const int r0 = warp * 16;
    const float scale = rsqrtf(static_cast<float>(HD));
    // key block j's K, V in buffer j & 1; block j + 1 is copied in while j computes
    auto kv_issue = [&](int j) {
        __nv_bfloat16* kb = Qs + M::ROW * (1 + 2 * (j & 1));
        const int kk0 = j * kMBlk;
        load_rows_async<HD>(kb, qkv, ld, b.row0 + kk0, min(kMBlk, b.len - kk0), (H + kvh) * HD);
        load_rows_async<HD>(kb + M::ROW, qkv, ld, b.row0 + kk0, min(kMBlk, b.len - kk0), (H + KV + kvh) * HD);
        cp_async_commit();
    };
    load_rows_async<HD>(Qs, qkv, ld, b.row0 + b.q0, nq, h * HD);
    kv_issue(0);
    float o[HD / 8][4];
#pragma unroll
    for (int dt = 0; dt < HD / 8; ++dt)
#pragma unroll
        for (int c = 0; c < 4; ++c) o[dt][c] = 0.f;
    float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
    const int nblk = (b.q0 + nq + kMBlk - 1) / kMBlk;
    for (int j = 0; j < nblk; ++j) {
        const int k0 = j * kMBlk;
        const int nk = min(kMBlk, b.len - k0);
        if (j + 1 < nblk) {
            kv_issue(j + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const __nv_bfloat16* Ks = Qs + M::ROW * (1 + 2 * (j & 1));
        const __nv_bfloat16* Vs = Ks + M::ROW;
        float s[8][4];
        qk_tile<HD>(s, Qs, r0, Ks, g, tq);
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int row = r0 + g + (c >= 2 ? 8 : 0), key = nt * 8 + 2 * tq + (c & 1);
                const bool ok = key < nk && row < nq && k0 + key <= b.q0 + row;
                s[nt][c] = ok ? s[nt][c] * scale : -INFINITY;
                mx[c >> 1] = fmaxf(mx[c >> 1], s[nt][c]);
            }
        float corr[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 1));
            mx[i] = fmaxf(mx[i], __shfl_xor_sync(0xffffffffu, mx[i], 2));
            const float mn = fmaxf(m[i], mx[i]);
            corr[i] = m[i] == -INFINITY ? 0.f : __expf(m[i] - mn);
            m[i] = mn;
        }
        float rs[2] = {0.f, 0.f};
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float mi = m[c >> 1];
                const float p = mi == -INFINITY ? 0.f : __expf(s[nt][c] - mi);
                s[nt][c] = p;
                rs[c >> 1] += p;
            }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], 1);
            rs[i] += __shfl_xor_sync(0xffffffffu, rs[i], 2);
            l[i] = l[i] * corr[i] + rs[i];
        }
#pragma unroll
        for (int dt = 0; dt < HD / 8; ++dt) {
            o[dt][0] *= corr[0];
            o[dt][1] *= corr[0];
            o[dt][2] *= corr[1];
            o[dt][3] *= corr[1];
        }
        pv_tile<HD>(o, s, Vs, lane);
        __syncthreads();  // buffer j & 1 is refilled by iteration j + 1's copy of block j + 2
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int row = r0 + g + 8 * i;
        if (row >= nq) continue;
        const size_t r = static_cast<size_t>(b.row0 + b.q0 + row);
        const float inv = l[i] > 0.f ? 1.f / l[i] : 0.f;
#pragma unroll
        for (int dt = 0; dt < HD / 8; ++dt)
            *reinterpret_cast<uint32_t*>(out + r * (H * HD) + h * HD + dt * 8 + 2 * tq) =
                pack_bf16(o[dt][2 * i] * inv, o[dt][2 * i + 1] * inv);
        if (tq == 0) lse[r * H + h] = m[i] + logf(l[i]);
    }
}

template <int HD>
__global__ void __launch_bounds__(128) attn_dq_mma(const TBlk* __restrict__ blks, const __nv_bfloat16* __restrict__ qkv,
                                                   int ld, int H, int KV, const __nv_bfloat16* __restrict__ dout,
                                                   const float* __restrict__ lse, const float* __restrict__ dvec,
                                                   float* __restrict__ dqkv, int ldd, float theta) {
    using M = MmaT<HD>;
    extern __shared__ __align__(16) uint8_t smraw[];
    __nv_bfloat16* Qs = reinterpret_cast<__nv_bfloat16*>(smraw);
    __nv_bfloat16* dOs = Qs + M::ROW;
    const TBlk b = blks[blockIdx.x];
    const int h = blockIdx.y, kvh = h / (H / KV);
    const int nq = min(kMBlk, b.len - b.q0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
    const int r0 = warp * 16;
    const float scale = rsqrtf(static_cast<float>(HD));
    auto kv_issue = [&](int j) {  // key block j's K, V into buffer j & 1
        __nv_bfloat16* kb = Qs + M::ROW * (2 + 2 * (j & 1));
        const int kk0 = j * kMBlk;
        load_rows_async<HD>(kb, qkv, ld, b.row0 + kk0, min(kMBlk, b.len - kk0), (H + kvh) * HD);
        load_rows_async<HD>(kb + M::ROW, qkv, ld, b.row0 + kk0, min(kMBlk, b.len - kk0), (H + KV + kvh) * HD);
        cp_async_commit();
    };
    load_rows_async<HD>(Qs, qkv, ld, b.row0 + b.q0, nq, h * HD);
    load_rows_async<HD>(dOs, dout, static_cast<size_t>(H) * HD, b.row0 + b.q0, nq, h * HD);
    kv_issue(0);
    float lr[2], dr[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int row = min(r0 + g + 8 * i, nq - 1);
        const size_t r = static_cast<size_t>(b.row0 + b.q0 + row);
        lr[i] = lse[r * H + h];
        dr[i] = dvec[r * H + h];
    }
    float dq[HD / 8][4];
#pragma unroll
    for (int dt = 0; dt < HD / 8; ++dt)
#pragma unroll
        for (int c = 0; c < 4; ++c) dq[dt][c] = 0.f;
    const int nblk = (b.q0 + nq + kMBlk - 1) / kMBlk;
    for (int j = 0; j < nblk; ++j) {
        const int k0 = j * kMBlk;
        const int nk = min(kMBlk, b.len - k0);
        if (j + 1 < nblk) {
            kv_issue(j + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const __nv_bfloat16* Ks = Qs + M::ROW * (2 + 2 * (j & 1));
        const __nv_bfloat16* Vs = Ks + M::ROW;
        float s[8][4], dp[8][4];
        qk_tile<HD>(s, Qs, r0, Ks, g, tq);    // S = Q K^T
        qk_tile<HD>(dp, dOs, r0, Vs, g, tq);  // dP = dO V^T
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int i = c >> 1;
                const int row = r0 + g + 8 * i, key = nt * 8 + 2 * tq + (c & 1);
                const bool ok = key < nk && row < nq && k0 + key <= b.q0 + row;
                const float p = ok ? __expf(s[nt][c] * scale - lr[i]) : 0.f;
                s[nt][c] = p * (dp[nt][c] - dr[i]);  // dS
            }
        pv_tile<HD>(dq, s, Ks, lane);  // dQ += dS K
        __syncthreads();  // buffer j & 1 is refilled by iteration j + 1's copy of block j + 2
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int row = r0 + g + 8 * i;
        if (row >= nq) continue;
        const size_t r = static_cast<size_t>(b.row0 + b.q0 + row);
        if (theta > 0.f) rope_bwd_frag<HD>(dq, i, tq, b.q0 + row, theta);  // d q_pre-RoPE
#pragma unroll
        for (int dt = 0; dt < HD / 8; ++dt) {
            float2 v = make_float2(dq[dt][2 * i] * scale, dq[dt][2 * i + 1] * scale);
            *reinterpret_cast<float2*>(dqkv + r * ldd + h * HD + dt * 8 + 2 * tq) = v;
        }
    }
}

// gsplit > 1: the G query heads of a KV head are split over gsplit CTAs
// (blockIdx.y = kvh * gsplit + part); each writes its dK / dV sums into
// part[gs][row][2 * KV * HD] and dkv_combine adds them in part order
// (deterministic).  The first key block of a long sequence otherwise walks
// G x (its query blocks) tiles alone and sets the kernel's duration.
template <int HD>
__global__ void __launch_bounds__(128) attn_dkv_mma(const TBlk* __restrict__ blks, const __nv_bfloat16* __restrict__ qkv,
                                                    int ld, int H, int KV, const __nv_bfloat16* __restrict__ dout,
                                                    const float* __restrict__ lse, const float* __restrict__ dvec,
                                                    float* __restrict__ dqkv, int ldd, int gsplit, float* __restrict__ part,
                                                    int rows, float theta) {
    using M = MmaT<HD>;
    extern __shared__ __align__(16) uint8_t smraw[];
    __nv_bfloat16* Ks = reinterpret_cast<__nv_bfloat16*>(smraw);
    __nv_bfloat16* Vs = Ks + M::ROW;
    // double-buffered (Q, dO) tiles [2][2][ROW] and (lse, dvec) rows [2][2][kMBlk]
    __nv_bfloat16* QdO = Vs + M::ROW;
    float* ld_s = reinterpret_cast<float*>(QdO + 4 * M::ROW);
    const TBlk b = blks[blockIdx.x];  // q0 = key block start
    const int kvh = blockIdx.y / gsplit, gs = blockIdx.y % gsplit, G = H / KV;
    const int gh0 = gs * G / gsplit, gh1 = (gs + 1) * G / gsplit;
    const int k0 = b.q0, nk = min(kMBlk, b.len - k0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
    const int r0 = warp * 16;  // this warp's 16 keys
    const float scale = rsqrtf(static_cast<float>(HD));
    // iterations it = (head, query block) pairs; iteration it + 1's tiles are
    // copied in (cp.async) while it computes
    const int nqb = (b.len - k0 + kMBlk - 1) / kMBlk, n_it = (gh1 - gh0) * nqb;
    auto qd_issue = [&](int it) {
        const int h = kvh * G + gh0 + it / nqb, q0 = k0 + (it % nqb) * kMBlk, nq = min(kMBlk, b.len - q0);
        __nv_bfloat16* qb = QdO + 2 * M::ROW * (it & 1);
        load_rows_async<HD>(qb, qkv, ld, b.row0 + q0, nq, h * HD);
        load_rows_async<HD>(qb + M::ROW, dout, static_cast<size_t>(H) * HD, b.row0 + q0, nq, h * HD);
        cp_async_commit();
        float* lb = ld_s + 2 * kMBlk * (it & 1);
        for (int i = threadIdx.x; i < kMBlk; i += blockDim.x) {
            const size_t r = static_cast<size_t>(b.row0 + q0 + min(i, nq - 1));
            lb[i] = lse[r * H + h];
            lb[kMBlk + i] = dvec[r * H + h];
        }
    };
    load_rows_async<HD>(Ks, qkv, ld, b.row0 + k0, nk, (H + kvh) * HD);
    load_rows_async<HD>(Vs, qkv, ld, b.row0 + k0, nk, (H + KV + kvh) * HD);
    if (n_it > 0) qd_issue(0);
    float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
    for (int dt = 0; dt < HD / 8; ++dt)
#pragma unroll
        for (int c = 0; c < 4; ++c) dk[dt][c] = dv[dt][c] = 0.f;
    for (int it = 0; it < n_it; ++it) {
        {
            const int q0 = k0 + (it % nqb) * kMBlk;
            const int nq = min(kMBlk, b.len - q0);
            if (it + 1 < n_it) {
                qd_issue(it + 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            const __nv_bfloat16* Qs = QdO + 2 * M::ROW * (it & 1);
            const __nv_bfloat16* dOs = Qs + M::ROW;
            const float* lse_s = ld_s + 2 * kMBlk * (it & 1);
            const float* d_s = lse_s + kMBlk;
            float st[8][4], dpt[8][4];
            qk_tile<HD>(st, Ks, r0, Qs, g, tq);   // S^T = K Q^T   (keys x queries)
            qk_tile<HD>(dpt, Vs, r0, dOs, g, tq); // dP^T = V dO^T
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int key = r0 + g + (c >= 2 ? 8 : 0), qi = nt * 8 + 2 * tq + (c & 1);
                    const bool ok = qi < nq && key < nk && k0 + key <= q0 + qi;
                    const float p = ok ? __expf(st[nt][c] * scale - lse_s[qi]) : 0.f;
                    st[nt][c] = p;
                    dpt[nt][c] = p * (dpt[nt][c] - d_s[qi]);  // dS^T
                }
            pv_tile<HD>(dv, st, dOs, lane);  // dV += P^T dO
            pv_tile<HD>(dk, dpt, Qs, lane);  // dK += dS^T Q
            __syncthreads();  // buffer it & 1 is refilled by iteration it + 1's copy of it + 2
        }
    }
    if (n_it == 0) cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int key = r0 + g + 8 * i;
        if (key >= nk) continue;
        const size_t r = static_cast<size_t>(b.row0 + k0 + key);
        if (theta > 0.f) rope_bwd_frag<HD>(dk, i, tq, k0 + key, theta);  // linear: partial sums commute
        // gsplit == 1: straight into dqkv's K | V columns; else this part's row
        float* dst = gsplit == 1 ? dqkv + r * ldd + H * HD
                                 : part + (static_cast<size_t>(gs) * rows + r) * (2 * KV * HD);
#pragma unroll
        for (int dt = 0; dt < HD / 8; ++dt) {
            *reinterpret_cast<float2*>(dst + kvh * HD + dt * 8 + 2 * tq) =
                make_float2(dk[dt][2 * i] * scale, dk[dt][2 * i + 1] * scale);
            *reinterpret_cast<float2*>(dst + (KV + kvh) * HD + dt * 8 + 2 * tq) =
                make_float2(dv[dt][2 * i], dv[dt][2 * i + 1]);
        }
    }
}

// dqkv[r][H*HD + c] = sum over parts (in order) of part[p][r][c], c < w = 2*KV*HD
static __global__ void dkv_combine(const float* __restrict__ part, int parts, int rows, int w, float* __restrict__ dqkv,
                                   int ldd, int col0) {
    const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * 4;
    if (i >= static_cast<int64_t>(rows) * w) return;
    const int64_t r = i / w, c = i % w;
    float4 acc = *reinterpret_cast<const float4*>(part + i);
    for (int p = 1; p < parts; ++p) {
        const float4 v = *reinterpret_cast<const float4*>(part + static_cast<size_t>(p) * rows * w + i);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
    }
    *reinterpret_cast<float4*>(dqkv + r * ldd + col0 + c) = acc;
}

}  // namespace train
}  // namespace oppo
