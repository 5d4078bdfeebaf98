// attn_dec.cuh — the actor's decode attention with RoPE and the paged KV
// append fused in (bf16).  One CTA of 4 warps per (decode row, KV head
// [, split]):
//   1. assemble this KV group's slice of the qkv row — the G query heads, k
//      and v — from the decode GEMM's split-K partials (+ bias, rounded to
//      bf16 exactly as a stored qkv row) or from a bf16 qkv row; apply RoPE
//      (rotate-half, same arithmetic as rope_append) to q and k;
//   2. the CTA whose position range holds the new token writes k, v into the
//      paged cache;
//   3. the 4 warps split the context positions (tiles of TP, double-buffered
//      cp.async per warp) and run S = QK^T / online softmax / O += PV on
//      mma.sync m16n8k16 with the G query heads stacked as MMA rows, so each
//      K/V tile is read from HBM once for the whole group;
//   4. the 4 warp partials (and, for split-KV clusters, every CTA's partials
//      pushed into rank 0 through DSMEM) are merged in shared memory.
// Replaces rope_append + attn_mma<HD,1> (+ split combine) on the decode path:
// one launch per layer instead of two, no qkv/q round trip through HBM.
#pragma once

#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include "attn_mma.cuh"
#include "common.cuh"
#include "model.cuh"

namespace oppo {

template <int HD, int NW = 4, int TPO = 0>
struct AttnDecCfg {
    static constexpr int WARPS = NW;
    static constexpr int THREADS = 32 * NW;
    // positions per warp tile (8 warps: half-size tiles, same shared memory;
    // TPO = 16 with 4 warps: half the shared memory, more resident CTAs)
    static constexpr int TP = TPO ? TPO : ((HD >= 128 || NW == 8) ? 16 : 32);
    static constexpr int LDS = HD + 8;              // padded smem row (elements)
    static constexpr int WARP_BYTES = 2 * 2 * TP * LDS * 2;  // K,V double buffer
    static constexpr int SLOT = 16 * HD + 32;                // merge partial (floats)
    static constexpr int QBYTES = 16 * LDS * 2;
    // fp32 q/k/v staging of phase 1 (own region: the first K/V tiles load meanwhile)
    static constexpr int FQ_BYTES = 18 * HD * 4;
    static constexpr int SMEM = NW * WARP_BYTES + QBYTES + FQ_BYTES;  // early-tile launch
    static constexpr int SMEM_ALIAS = NW * WARP_BYTES + QBYTES;       // staging aliases K/V
    static_assert(NW * WARP_BYTES >= FQ_BYTES, "q/k/v staging must fit the K/V buffers");
    static_assert(NW * WARP_BYTES >= NW * (16 * HD + 32) * 4, "warp partials must fit the K/V buffers");
    // CTAs of a split-KV cluster whose 4 x nsp partials fit rank 0's K/V buffers
    static constexpr int MAX_SPLIT = (NW * WARP_BYTES) / (NW * SLOT * 4) > 8 ? 8
                                                                              : (NW * WARP_BYTES) / (NW * SLOT * 4);
};

template <int HD, int NW, int TPO = 0>
__global__ void __launch_bounds__(32 * NW)
    attn_dec(const float* __restrict__ part, int n_part, size_t part_stride,
             const float* __restrict__ bias, const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* out,
             KvView kv, int layer, int n_heads, const int32_t* __restrict__ slot_r,
             const int32_t* __restrict__ pos_r, int rows, float theta, int early_tiles, int minpos) {
    using namespace am;
    using Cf = AttnDecCfg<HD, NW, TPO>;
    constexpr int TP = Cf::TP, LDS = Cf::LDS, NT = TP / 8, DT = HD / 8, NTH = Cf::THREADS;
    extern __shared__ __align__(128) uint8_t adsm[];
    uint8_t* kvbuf = adsm;                                                     // 4 warps x K/V x 2
    auto sQ = reinterpret_cast<__nv_bfloat16(*)[LDS]>(adsm + NW * Cf::WARP_BYTES);  // [16][LDS]
    // [G+2][HD] fp32 staging: its own region when the first tiles load early,
    // else aliased onto the (still idle) K/V buffers (smaller launch footprint)
    float* fq = reinterpret_cast<float*>(early_tiles ? adsm + NW * Cf::WARP_BYTES + Cf::QBYTES : adsm);
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x;
    if (r >= rows) return;  // whole cluster (same r) leaves together
    const int h = blockIdx.y, KV = kv.kv_heads, G = n_heads / KV, H = n_heads;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int slot = slot_r[r], pos = pos_r[r], ctx = pos + 1;
    const int nsp = gridDim.z, z = blockIdx.z;
    // this row's split count: at least minpos positions per split (a short
    // context stays in one CTA; the cluster's other CTAs get empty ranges and
    // only take part in the merge with m = -inf, l = 0)
    const int want = max(1, min(nsp, (ctx + minpos - 1) / minpos));
    const int slen = (ctx + want - 1) / want;
    const int p_begin = min(ctx, z * slen), p_end = min(ctx, p_begin + slen);
    const bool owner = pos >= p_begin && pos < p_end;  // this CTA appends the new k, v

    // K/V tiles of positions before the new token do not depend on this
    // iteration: each warp issues its first tile now, so the loads overlap the
    // qkv fold / RoPE / append below (a tile holding `pos` waits for the append)
    const int lane_ = tid & 31;
    auto sK = reinterpret_cast<__nv_bfloat16(*)[TP][LDS]>(kvbuf + warp * Cf::WARP_BYTES);
    auto sV = reinterpret_cast<__nv_bfloat16(*)[TP][LDS]>(kvbuf + warp * Cf::WARP_BYTES + 2 * TP * LDS * 2);
    const __nv_bfloat16* kc = static_cast<const __nv_bfloat16*>(kv.k);
    const __nv_bfloat16* vc = static_cast<const __nv_bfloat16*>(kv.v);
    auto load_tile = [&](int buf, int t0) {
        constexpr int CHUNKS = TP * HD / 8;  // 16-byte chunks per tensor
#pragma unroll
        for (int c = lane_; c < CHUNKS; c += 32) {
            const int p = c / (HD / 8), e = (c % (HD / 8)) * 8;
            const int ps = t0 + p;
            const bool valid = ps < p_end;
            const size_t base = valid ? kv_index<__nv_bfloat16>(kv, layer, slot, ps, h) + e : 0;
            cp_async16(&sK[buf][p][e], kc + base, valid);
            cp_async16(&sV[buf][p][e], vc + base, valid);
        }
        cp_async_commit();
    };
    const int first = p_begin + warp * TP;
    const bool early = early_tiles && first < p_end && first + TP <= pos;
    if (early) load_tile(0, first);

    // ---- 1. q (G heads), k, v of this KV group: fold partials, bias, bf16 round
    const int width = (H + 2 * KV) * HD;
    const int nvals = (G + 2) * HD;
    for (int i = tid; i < nvals; i += NTH) {
        const int gi = i / HD, d = i % HD;
        const int col = gi < G ? (h * G + gi) * HD + d : gi == G ? (H + h) * HD + d : (H + KV + h) * HD + d;
        float v;
        if (part) {  // split loads issued 4 at a time (one memory round trip per 4 splits)
            float a = 0.f;
            const float* p = part + static_cast<size_t>(r) * width + col;
            for (int s0 = 0; s0 < n_part; s0 += 8) {  // 8 split loads in flight, split order
                float pv[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) pv[k] = s0 + k < n_part ? __ldcg(p + (s0 + k) * part_stride) : 0.f;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (s0 + k >= n_part) break;
                    a += pv[k];
                }
            }
            v = tof(fromf<__nv_bfloat16>(a + (bias ? bias[col] : 0.f)));
        } else {
            v = tof(qkv[static_cast<size_t>(r) * width + col]);
        }
        fq[gi * HD + d] = v;
    }
    __syncthreads();
    // RoPE on q heads and k (rotate-half), then q -> sQ (bf16), new k/v -> cache
    const int half = HD / 2;
    for (int i = tid; i < (G + 1) * half; i += NTH) {
        const int gi = i / half, d = i % half;
        const float inv_freq = __powf(theta, -2.0f * d / HD);
        float sn, cs;
        sincosf(pos * inv_freq, &sn, &cs);
        const float x1 = fq[gi * HD + d], x2 = fq[gi * HD + d + half];
        const float y1 = x1 * cs - x2 * sn, y2 = x2 * cs + x1 * sn;
        if (gi < G) {
            sQ[gi][d] = fromf<__nv_bfloat16>(y1);
            sQ[gi][d + half] = fromf<__nv_bfloat16>(y2);
        } else if (owner) {
            __nv_bfloat16* kc = static_cast<__nv_bfloat16*>(kv.k) + kv_index<__nv_bfloat16>(kv, layer, slot, pos, h);
            kc[d] = fromf<__nv_bfloat16>(y1);
            kc[d + half] = fromf<__nv_bfloat16>(y2);
        }
    }
    if (owner) {
        __nv_bfloat16* vc = static_cast<__nv_bfloat16*>(kv.v) + kv_index<__nv_bfloat16>(kv, layer, slot, pos, h);
        for (int d = tid; d < HD; d += NTH) vc[d] = fromf<__nv_bfloat16>(fq[(G + 1) * HD + d]);
    }
    for (int i = tid; i < (16 - G) * HD; i += NTH) sQ[G + i / HD][i % HD] = fromf<__nv_bfloat16>(0.f);
    __threadfence_block();
    __syncthreads();  // q in smem; the appended k/v visible to this CTA's tile loads

    // ---- 2. per-warp flash attention over tiles w, w+4, ... of [p_begin, p_end)
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
    const float scale = rsqrtf(static_cast<float>(HD)) * 1.4426950408889634f;  // exp2 domain
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    float o[DT][4];
#pragma unroll
    for (int d = 0; d < DT; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.f;
    int buf = 0;
    if (!early && first < p_end) load_tile(0, first);
    for (int t0 = first; t0 < p_end; t0 += NW * TP) {
        if (t0 + NW * TP < p_end) {
            load_tile(buf ^ 1, t0 + NW * TP);
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
        __syncwarp();  // the buffer is refilled two tiles later
        buf ^= 1;
    }
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);

    // ---- 3. merge 4 warps x nsp CTAs: partial slot (z * 4 + warp) of rank 0
    namespace cg = cooperative_groups;
    float* dst;
    if (nsp > 1) {
        cg::cluster_group cl = cg::this_cluster();
        cl.sync();  // every rank (incl. 0) is done with its K/V buffers
        dst = cl.map_shared_rank(reinterpret_cast<float*>(kvbuf), 0);
    } else {
        __syncthreads();
        dst = reinterpret_cast<float*>(kvbuf);
    }
    dst += (z * NW + warp) * Cf::SLOT;
#pragma unroll
    for (int d = 0; d < DT; ++d) {
        const int c = d * 8 + tig * 2;
        *reinterpret_cast<float2*>(dst + row0 * HD + c) = make_float2(o[d][0], o[d][1]);
        *reinterpret_cast<float2*>(dst + row1 * HD + c) = make_float2(o[d][2], o[d][3]);
    }
    if (tig == 0) {
        *reinterpret_cast<float2*>(dst + 16 * HD + row0 * 2) = make_float2(m0, l0);
        *reinterpret_cast<float2*>(dst + 16 * HD + row1 * 2) = make_float2(m1, l1);
    }
    if (nsp > 1) {
        cg::this_cluster().sync();
        if (z != 0) return;
    } else {
        __syncthreads();
    }
    const float* bufm = reinterpret_cast<const float*>(kvbuf);
    const int np = NW * nsp;
    for (int e = tid; e < G * HD; e += NTH) {
        const int g = e / HD, c = e % HD;
        float mx = -INFINITY;
        for (int sp = 0; sp < np; ++sp) mx = fmaxf(mx, bufm[sp * Cf::SLOT + 16 * HD + g * 2]);
        float L = 0.f, O = 0.f;
        for (int sp = 0; sp < np; ++sp) {
            const float ms = bufm[sp * Cf::SLOT + 16 * HD + g * 2];
            const float wgt = ms == -INFINITY ? 0.f : exp2f(ms - mx);
            L += bufm[sp * Cf::SLOT + 16 * HD + g * 2 + 1] * wgt;
            O += bufm[sp * Cf::SLOT + e] * wgt;
        }
        out[(static_cast<size_t>(r) * H + h * G + g) * HD + c] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
    }
}

}  // namespace oppo
