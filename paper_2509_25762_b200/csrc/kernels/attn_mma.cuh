// attn_mma.cuh — bf16 GQA attention over the paged KV cache on tensor cores
// (mma.sync m16n8k16, fp32 accumulation), used for both decode and chunked
// prefill.
//
// A CTA owns one KV head of one slot and 16*WARPS "rows" = (query, q-head)
// pairs: the G query heads that share the KV head are stacked as rows, so
// every K/V tile is read from HBM once for all of them.  K/V tiles of 64
// positions are staged in shared memory with cp.async (double-buffered,
// zero-filled past the context); S = Q K^T takes K fragments via ldmatrix,
// P V takes V fragments via ldmatrix.trans; the running softmax is the usual
// flash-attention recurrence on the accumulator fragments.
//   decode : WARPS = 1, one query row per CTA, grid.z = split-KV chunks; the
//            split CTAs of a row form one thread-block cluster and rank 0
//            merges the partials through distributed shared memory (no
//            workspace round trip, no combine kernel; ws_o == nullptr);
//            with ws_o set, partials go to the workspace instead and
//            attn_split_combine merges them.
//   prefill: WARPS = 4, a query block of one slot (QBlock), causal mask.
#pragma once

#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "model.cuh"

namespace oppo {

namespace am {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_addr(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_addr(p)));
}
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

}  // namespace am

// largest split-KV cluster whose partials fit the K/V buffers of rank 0
template <int HD>
constexpr int attn_merge_splits() {
    constexpr int TP = HD >= 128 ? 32 : 64, LDS = HD + 8;
    constexpr int n = (2 * 2 * TP * LDS * 2) / ((16 * HD + 32) * 4);
    return n > 8 ? 8 : n;
}

template <int HD, int WARPS>
__global__ void __launch_bounds__(32 * WARPS)
    attn_mma(const __nv_bfloat16* __restrict__ q, __nv_bfloat16* out, KvView kv, int layer,
             int n_heads, const int32_t* __restrict__ slot_r, const int32_t* __restrict__ pos_r,
             int rows, float* ws_o, float* ws_ml, const QBlock* __restrict__ blocks) {
    using namespace am;
    constexpr int TP = HD >= 128 ? 32 : 64;  // positions per KV tile (static smem < 48 KB)
    constexpr int LDS = HD + 8;  // padded smem row (elements): conflict-free ldmatrix
    constexpr int NT = TP / 8;   // score n-tiles per KV tile
    constexpr int DT = HD / 8;   // output n-tiles
    // K/V double buffers; after the loop the same bytes hold the split-KV
    // merge buffer of the cluster's rank 0 (kMergeSplits partials)
    __shared__ __align__(128) uint8_t smraw[2 * 2 * TP * LDS * 2];
    auto sK = reinterpret_cast<__nv_bfloat16(*)[TP][LDS]>(smraw);
    auto sV = reinterpret_cast<__nv_bfloat16(*)[TP][LDS]>(smraw + 2 * TP * LDS * 2);
    pdl_trigger();
    pdl_wait();

    const int G = n_heads / kv.kv_heads;
    const int h = blockIdx.y;
    int slot, qpos0, nq;
    size_t qrow0;
    int p_begin = 0, p_end;
    if (blocks) {
        const QBlock b = blocks[blockIdx.x];
        slot = b.slot;
        qpos0 = b.pos0;
        nq = b.n;
        qrow0 = b.row0;
        p_end = qpos0 + nq;
    } else {
        const int r = blockIdx.x;
        if (r >= rows) return;
        slot = slot_r[r];
        qpos0 = pos_r[r];
        nq = 1;
        qrow0 = r;
        const int ctx = qpos0 + 1, nsp = gridDim.z;
        const int slen = (ctx + nsp - 1) / nsp;
        p_begin = blockIdx.z * slen;
        p_end = min(ctx, p_begin + slen);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
    // the two rows this thread accumulates: (query, head) = divmod(row, G)
    const int row0 = warp * 16 + gid, row1 = row0 + 8;
    const int qi0 = row0 / G, g0 = row0 % G, qi1 = row1 / G, g1 = row1 % G;
    const bool ok0 = qi0 < nq, ok1 = qi1 < nq;
    const int qp0 = qpos0 + qi0, qp1 = qpos0 + qi1;

    // Q fragments (A operand, rows = (query, head))
    uint32_t qf[HD / 16][4];
    {
        const __nv_bfloat16* q0 = q + ((qrow0 + (ok0 ? qi0 : 0)) * n_heads + h * G + g0) * HD;
        const __nv_bfloat16* q1 = q + ((qrow0 + (ok1 ? qi1 : 0)) * n_heads + h * G + g1) * HD;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
            const int c = kk * 16 + tig * 2;
            qf[kk][0] = ok0 ? *reinterpret_cast<const uint32_t*>(q0 + c) : 0u;
            qf[kk][1] = ok1 ? *reinterpret_cast<const uint32_t*>(q1 + c) : 0u;
            qf[kk][2] = ok0 ? *reinterpret_cast<const uint32_t*>(q0 + c + 8) : 0u;
            qf[kk][3] = ok1 ? *reinterpret_cast<const uint32_t*>(q1 + c + 8) : 0u;
        }
    }
    const float scale = rsqrtf(static_cast<float>(HD)) * 1.4426950408889634f;  // exp2 domain
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    float o[DT][4];
#pragma unroll
    for (int d = 0; d < DT; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.f;

    const __nv_bfloat16* kc = static_cast<const __nv_bfloat16*>(kv.k);
    const __nv_bfloat16* vc = static_cast<const __nv_bfloat16*>(kv.v);
    auto load_tile = [&](int buf, int t0) {
        constexpr int CHUNKS = TP * HD / 8;  // 16-byte chunks per tensor
        for (int c = threadIdx.x; c < CHUNKS; c += 32 * WARPS) {
            const int p = c / (HD / 8), e = (c % (HD / 8)) * 8;
            const int pos = t0 + p;
            const bool valid = pos < p_end;
            const size_t base = valid ? kv_index<__nv_bfloat16>(kv, layer, slot, pos, h) + e : 0;
            cp_async16(&sK[buf][p][e], kc + base, valid);
            cp_async16(&sV[buf][p][e], vc + base, valid);
        }
        cp_async_commit();
    };
    int buf = 0;
    if (p_begin < p_end) load_tile(0, p_begin);
    for (int t0 = p_begin; t0 < p_end; t0 += TP) {
        if (t0 + TP < p_end) {
            load_tile(buf ^ 1, t0 + TP);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        // ---- S = Q K^T
        float s[NT][4];
#pragma unroll
        for (int j = 0; j < NT; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
            for (int j = 0; j < NT; j += 2) {
                // matrices: (tile j, dims kk*16..+7), (j, +8), (j+1, kk*16), (j+1, +8)
                const int mi = lane >> 3, r = lane & 7;
                uint32_t b[4];
                ldsm_x4(b, &sK[buf][(j + (mi >> 1)) * 8 + r][kk * 16 + (mi & 1) * 8]);
                mma16816(s[j], qf[kk], b[0], b[1]);
                mma16816(s[j + 1], qf[kk], b[2], b[3]);
            }
        }
        // ---- mask + online softmax (rows row0: s[.][0..1], row1: s[.][2..3])
        float mx0 = m0, mx1 = m1;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int pos = t0 + j * 8 + tig * 2 + (c & 1);
                const bool r1 = c >= 2;
                const bool ok = pos < p_end && pos <= (r1 ? qp1 : qp0) && (r1 ? ok1 : ok0);
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
        uint32_t pa[NT / 2][4];  // P as A fragments (two score tiles per k=16 block)
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
        // ---- O += P V
#pragma unroll
        for (int kk = 0; kk < NT / 2; ++kk) {
#pragma unroll
            for (int d = 0; d < DT; d += 2) {
                // matrices: (pos kk*16..+7, dims d*8), (pos +8, d*8), (pos kk*16, (d+1)*8), (pos +8, (d+1)*8)
                const int mi = lane >> 3, r = lane & 7;
                uint32_t b[4];
                ldsm_x4_t(b, &sV[buf][kk * 16 + (mi & 1) * 8 + r][(d + (mi >> 1)) * 8]);
                mma16816(o[d], pa[kk], b[0], b[1]);
                mma16816(o[d + 1], pa[kk], b[2], b[3]);
            }
        }
        __syncthreads();  // the buffer is refilled two tiles later
        buf ^= 1;
    }
    // ---- finalize: row sums across the quad, normalise, store
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
    if (blocks || gridDim.z == 1) {
        const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
#pragma unroll
        for (int d = 0; d < DT; ++d) {
            const int c = d * 8 + tig * 2;
            if (ok0)
                *reinterpret_cast<uint32_t*>(out + ((qrow0 + qi0) * n_heads + h * G + g0) * HD + c) =
                    pack_bf16(o[d][0] * i0, o[d][1] * i0);
            if (ok1)
                *reinterpret_cast<uint32_t*>(out + ((qrow0 + qi1) * n_heads + h * G + g1) * HD + c) =
                    pack_bf16(o[d][2] * i1, o[d][3] * i1);
        }
    } else if (!ws_o) {  // split-KV merge inside the cluster (DSMEM)
        // every rank pushes its unnormalised O rows and (max, sum) into rank
        // 0's shared memory with remote stores (no remote-load latency on the
        // merge), then rank 0 merges from local shared memory.
        namespace cg = cooperative_groups;
        cg::cluster_group cl = cg::this_cluster();
        const int nsp = static_cast<int>(cl.num_blocks()), rank = static_cast<int>(cl.block_rank());
        constexpr int SLOT = 16 * HD + 32;  // floats per split: O[16][HD], (m, l)[16]
        cl.sync();                          // rank 0 is done with its K/V buffers
        float* dst = cl.map_shared_rank(reinterpret_cast<float*>(smraw), 0) + rank * SLOT;
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
        cl.sync();  // release/acquire: the pushes are visible to rank 0
        if (rank == 0) {
            const float* buf = reinterpret_cast<const float*>(smraw);
            const int valid_rows = min(16, nq * G);
            for (int e = lane; e < valid_rows * HD; e += 32) {
                const int r = e / HD, c = e % HD;
                float mx = -INFINITY;
                for (int sp = 0; sp < nsp; ++sp) mx = fmaxf(mx, buf[sp * SLOT + 16 * HD + r * 2]);
                float L = 0.f, O = 0.f;
                for (int sp = 0; sp < nsp; ++sp) {
                    const float ms = buf[sp * SLOT + 16 * HD + r * 2];
                    const float wgt = ms == -INFINITY ? 0.f : exp2f(ms - mx);
                    L += buf[sp * SLOT + 16 * HD + r * 2 + 1] * wgt;
                    O += buf[sp * SLOT + e] * wgt;
                }
                const int qi = r / G, g = r % G;
                out[((qrow0 + qi) * n_heads + h * G + g) * HD + c] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
            }
        }
    } else {  // split-KV partial: unnormalised accumulator, running max (natural log domain), sum
        const int nsp = gridDim.z, sp = blockIdx.z;
        const float ln2 = 0.6931471805599453f;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const bool okh = half ? ok1 : ok0;
            if (!okh) continue;
            const int head = h * G + (half ? g1 : g0);
            const size_t oi = (static_cast<size_t>(qrow0) * n_heads + head) * nsp + sp;
#pragma unroll
            for (int d = 0; d < DT; ++d) {
                const int c = d * 8 + tig * 2;
                ws_o[oi * HD + c] = o[d][half * 2];
                ws_o[oi * HD + c + 1] = o[d][half * 2 + 1];
            }
            if (tig == 0) {
                const float mm = half ? m1 : m0;
                ws_ml[oi * 2] = mm == -INFINITY ? -INFINITY : mm * ln2;
                ws_ml[oi * 2 + 1] = half ? l1 : l0;
            }
        }
    }
}

}  // namespace oppo
