// model.cuh — non-GEMM kernels of the Qwen2-style decoder used by the actor,
// reward, critic and reference models (RMSNorm, RoPE, GQA, SwiGLU, q/k/v bias).
//
// Activations are token-major: one row per token of the current batch.  The
// residual stream is fp32; GEMM operands are T (bf16, or fp32 for parity).
// KV cache: per model and layer, K and V pools of pages laid out
// [page][kv_head][page_size][head_dim]; a slot's page table maps token
// position -> page.  Rows carry (slot, position, token) metadata.
#pragma once

#include "common.cuh"

namespace oppo {

struct RowMeta {          // one row of a batch (decode or prefill)
    int32_t* slot;        // [R]
    int32_t* pos;         // [R] cache position of the row's token
    int32_t* tok;         // [R] input token id
    int32_t* t;           // [R] response index of the row's *output* (pos - P + 2)
    uint64_t* key;        // [R] sampling key (decode rows)
};

// --------------------------------------------------------------- weights
// N(0, std) from the counter-based stream (seed, tensor id, index), Box-Muller.
template <class T>
__global__ void init_normal(T* w, int64_t n, uint64_t seed, uint64_t tensor, float std_) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint64_t h = mix64(seed ^ mix64(tensor * 0x9e3779b97f4a7c15ull + static_cast<uint64_t>(i)));
    const float u1 = (static_cast<float>(h >> 40) + 0.5f) * (1.0f / 16777216.0f);
    const float u2 = static_cast<float>((h >> 16) & 0xFFFFFFull) * (1.0f / 16777216.0f);
    const float z = sqrtf(-2.0f * logf(u1)) * cosf(6.283185307179586f * u2);
    w[i] = fromf<T>(z * std_);
}
template <class T>
__global__ void fill_value(T* w, int64_t n, float v) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) w[i] = fromf<T>(v);
}
template <class S, class D>
__global__ void convert(const S* s, D* d, int64_t n) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) d[i] = fromf<D>(tof(s[i]));
}

// ------------------------------------------------------------- embedding
template <class T>
__global__ void embed_rows(const T* __restrict__ emb, const int32_t* __restrict__ tok, float* x,
                           int rows, int d) {
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x;
    if (r >= rows) return;
    const T* src = emb + static_cast<size_t>(tok[r]) * d;
    float* dst = x + static_cast<size_t>(r) * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = tof(src[i]);
}

// ----------------------------------------------------------------- norms
// out[r] = x[r] * rsqrt(mean(x^2) + eps) * w; one warp per row.  Optionally
// also: head[r] = dot(out[r], hw) (value / reward head), and a copy of out[r]
// into a per-slot hidden cache at [slot][t] (for the PPO head update).
// With part != nullptr the row is first completed by the split-K partial sums
// of the preceding decode GEMM (gemm_dec DEC_PARTIAL): x[r] += sum_s part[s][r]
// in split order (deterministic), and the updated residual is written back.
template <class T>
__global__ void rmsnorm_rows(float* __restrict__ x, const float* __restrict__ w, T* out,
                             int rows, int d, float eps, const float* head_w, float* head_out,
                             T* cache, const int32_t* slot, const int32_t* tidx, int cache_rows,
                             int t_lo, int t_hi, const float* __restrict__ part, int n_part,
                             size_t part_stride) {
    pdl_trigger();
    pdl_wait();
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= rows) return;
    float* xr = x + static_cast<size_t>(warp) * d;
    // all of the row's float4 loads are issued before the reduction (one
    // memory round trip); d <= 32 * 4 * kMaxV4
    constexpr int kMaxV4 = 28;
    const int nv = d >> 2;
    float4 v[kMaxV4];
    float ss = 0.0f;
#pragma unroll
    for (int i = 0; i < kMaxV4; ++i) {
        const int c = lane + 32 * i;
        v[i] = c < nv ? reinterpret_cast<const float4*>(xr)[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (part) {
        for (int sp = 0; sp < n_part; ++sp) {
            const float4* pr = reinterpret_cast<const float4*>(part + sp * part_stride +
                                                               static_cast<size_t>(warp) * d);
#pragma unroll
            for (int i = 0; i < kMaxV4; ++i) {
                const int c = lane + 32 * i;
                if (c < nv) {
                    const float4 a = pr[c];
                    v[i].x += a.x;
                    v[i].y += a.y;
                    v[i].z += a.z;
                    v[i].w += a.w;
                }
            }
        }
#pragma unroll
        for (int i = 0; i < kMaxV4; ++i) {
            const int c = lane + 32 * i;
            if (c < nv) reinterpret_cast<float4*>(xr)[c] = v[i];
        }
    }
#pragma unroll
    for (int i = 0; i < kMaxV4; ++i) ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    ss = warp_sum(ss);
    const float inv = rsqrtf(ss / d + eps);
    float hd = 0.0f;
    T* orow = out ? out + static_cast<size_t>(warp) * d : nullptr;
    T* crow = nullptr;
    if (cache) {
        const int t = tidx[warp];
        if (t >= t_lo && t <= t_hi)
            crow = cache + (static_cast<size_t>(slot[warp]) * cache_rows + t) * d;
    }
#pragma unroll
    for (int i = 0; i < kMaxV4; ++i) {
        const int c = lane + 32 * i;
        if (c >= nv) break;
        const float4 g = __ldg(reinterpret_cast<const float4*>(w) + c);
        float y[4] = {v[i].x * inv * g.x, v[i].y * inv * g.y, v[i].z * inv * g.z, v[i].w * inv * g.w};
        __align__(8) T t4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) t4[k] = fromf<T>(y[k]);
        if constexpr (sizeof(T) == 2) {  // one 8-byte store per 4 values
            if (orow) *reinterpret_cast<uint2*>(orow + 4 * c) = *reinterpret_cast<const uint2*>(t4);
            if (crow) *reinterpret_cast<uint2*>(crow + 4 * c) = *reinterpret_cast<const uint2*>(t4);
        } else {
            if (orow) {
#pragma unroll
                for (int k = 0; k < 4; ++k) orow[4 * c + k] = t4[k];
            }
            if (crow) {
#pragma unroll
                for (int k = 0; k < 4; ++k) crow[4 * c + k] = t4[k];
            }
        }
        if (head_w) {
            const float4 hw = __ldg(reinterpret_cast<const float4*>(head_w) + c);
            hd += tof(t4[0]) * hw.x + tof(t4[1]) * hw.y + tof(t4[2]) * hw.z + tof(t4[3]) * hw.w;
        }
    }
    if (head_w) {
        hd = warp_sum(hd);
        if (lane == 0) head_out[warp] = hd;
    }
}

// Decode-path RMSNorm that first completes the residual row with the
// split-K partials of the preceding decode GEMM: x[r] += sum_s part[s][r]
// (split order, deterministic) and writes x back; then the same outputs as
// rmsnorm_rows (normed row, optional head dot and hidden-cache copy).  One
// 256-thread CTA per row, one float4 column per thread per pass, the split
// loads of a column issued together; gamma is fetched before the PDL wait.
template <class T>
__global__ void __launch_bounds__(256)
    residual_rmsnorm(float* __restrict__ x, const float* __restrict__ w, T* out, int rows, int d,
                     float eps, const float* __restrict__ part, int n_part, size_t part_stride,
                     const float* head_w, float* head_out, T* cache, const int32_t* slot,
                     const int32_t* tidx, int cache_rows, int t_lo, int t_hi) {
    constexpr int kCols = 4;  // float4 columns per thread: d <= 256 * 4 * 4
    const int r = blockIdx.x, tid = threadIdx.x, nv = d >> 2;
    float4 g[kCols], hw[kCols];
#pragma unroll
    for (int i = 0; i < kCols; ++i) {
        const int c = tid + 256 * i;
        g[i] = c < nv ? __ldg(reinterpret_cast<const float4*>(w) + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        hw[i] = (head_w && c < nv) ? __ldg(reinterpret_cast<const float4*>(head_w) + c)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    pdl_trigger();
    pdl_wait();
    if (r >= rows) return;
    float4* xr = reinterpret_cast<float4*>(x + static_cast<size_t>(r) * d);
    float4 v[kCols];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < kCols; ++i) {
        const int c = tid + 256 * i;
        if (c >= nv) continue;
        float4 a = xr[c];
        const float4* pc = reinterpret_cast<const float4*>(part) + static_cast<size_t>(r) * nv + c;
        const size_t ps = part_stride >> 2;
        for (int s0 = 0; s0 < n_part; s0 += 8) {  // 8 split loads in flight, summed in split order
            float4 pv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                pv[k] = s0 + k < n_part ? __ldcg(pc + (s0 + k) * ps) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (s0 + k >= n_part) break;
                a.x += pv[k].x; a.y += pv[k].y; a.z += pv[k].z; a.w += pv[k].w;
            }
        }
        if (n_part > 0) xr[c] = a;
        v[i] = a;
        ss += a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w;
    }
    __shared__ float red[8], red2[8];
    ss = warp_sum(ss);
    if ((tid & 31) == 0) red[tid >> 5] = ss;
    __syncthreads();
    ss = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) ss += red[i];
    const float inv = rsqrtf(ss / d + eps);
    T* orow = out ? out + static_cast<size_t>(r) * d : nullptr;
    T* crow = nullptr;
    if (cache) {
        const int t = tidx[r];
        if (t >= t_lo && t <= t_hi) crow = cache + (static_cast<size_t>(slot[r]) * cache_rows + t) * d;
    }
    float hd = 0.f;
#pragma unroll
    for (int i = 0; i < kCols; ++i) {
        const int c = tid + 256 * i;
        if (c >= nv) continue;
        const float y[4] = {v[i].x * inv * g[i].x, v[i].y * inv * g[i].y, v[i].z * inv * g[i].z,
                            v[i].w * inv * g[i].w};
        T t4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) t4[k] = fromf<T>(y[k]);
        if (orow) {
#pragma unroll
            for (int k = 0; k < 4; ++k) orow[4 * c + k] = t4[k];
        }
        if (crow) {
#pragma unroll
            for (int k = 0; k < 4; ++k) crow[4 * c + k] = t4[k];
        }
        if (head_w)
            hd += tof(t4[0]) * hw[i].x + tof(t4[1]) * hw[i].y + tof(t4[2]) * hw[i].z + tof(t4[3]) * hw[i].w;
    }
    if (head_w) {
        hd = warp_sum(hd);
        if ((tid & 31) == 0) red2[tid >> 5] = hd;
        __syncthreads();
        if (tid == 0) {
            float t = 0.f;
#pragma unroll
            for (int i = 0; i < 8; ++i) t += red2[i];
            head_out[r] = t;
        }
    }
}

// ------------------------------------------------- RoPE + paged KV append
// qkv row layout: [q (H*hd) | k (KV*hd) | v (KV*hd)], rotate-half RoPE.
// With part != nullptr the qkv row is assembled from the decode GEMM's
// split-K partials plus the q/k/v bias (rounded to T, exactly as the unsplit
// GEMM's bias epilogue stores it) into shared memory first.
template <class T>
__global__ void rope_append(const T* __restrict__ qkv, T* q_out, KvView kv, int layer,
                            const int32_t* __restrict__ slot, const int32_t* __restrict__ pos,
                            int rows, int n_heads, float theta, const float* __restrict__ part,
                            int n_part, size_t part_stride, const float* __restrict__ bias) {
    extern __shared__ uint8_t rope_smem[];
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x;
    if (r >= rows) return;
    const int hd = kv.head_dim, half = hd / 2;
    const int H = n_heads, KV = kv.kv_heads;
    const int width = (H + 2 * KV) * hd;
    const T* src = qkv + static_cast<size_t>(r) * width;
    if (part) {  // width % 4 == 0; float4 columns, split loads issued 4 at a time
        T* row = reinterpret_cast<T*>(rope_smem);
        const int nv = width >> 2;
        const size_t ps = part_stride >> 2;
        for (int c = threadIdx.x; c < nv; c += blockDim.x) {
            const float4* pc = reinterpret_cast<const float4*>(part) + static_cast<size_t>(r) * nv + c;
            float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
            int sp = 0;
            for (; sp + 4 <= n_part; sp += 4) {
                const float4 p0 = pc[sp * ps], p1 = pc[(sp + 1) * ps], p2 = pc[(sp + 2) * ps],
                             p3 = pc[(sp + 3) * ps];
                a.x += p0.x; a.y += p0.y; a.z += p0.z; a.w += p0.w;
                a.x += p1.x; a.y += p1.y; a.z += p1.z; a.w += p1.w;
                a.x += p2.x; a.y += p2.y; a.z += p2.z; a.w += p2.w;
                a.x += p3.x; a.y += p3.y; a.z += p3.z; a.w += p3.w;
            }
            for (; sp < n_part; ++sp) {
                const float4 p0 = pc[sp * ps];
                a.x += p0.x; a.y += p0.y; a.z += p0.z; a.w += p0.w;
            }
            const float4 b = bias ? reinterpret_cast<const float4*>(bias)[c] : make_float4(0.f, 0.f, 0.f, 0.f);
            row[4 * c] = fromf<T>(a.x + b.x);
            row[4 * c + 1] = fromf<T>(a.y + b.y);
            row[4 * c + 2] = fromf<T>(a.z + b.z);
            row[4 * c + 3] = fromf<T>(a.w + b.w);
        }
        __syncthreads();
        src = row;
    }
    const int p = pos[r], s = slot[r];
    T* kc = static_cast<T*>(kv.k);
    T* vc = static_cast<T*>(kv.v);
    // a thread keeps one rotary frequency d for the whole row (blockDim is a
    // multiple of hd/2): one sincos per thread instead of one per element
    const int d = threadIdx.x % half, hstep = blockDim.x / half;
    const float inv_freq = __powf(theta, -2.0f * d / hd);
    float sn, cs;
    sincosf(p * inv_freq, &sn, &cs);
    for (int head = threadIdx.x / half; head < H + KV; head += hstep) {
        const float x1 = tof(src[head * hd + d]);
        const float x2 = tof(src[head * hd + d + half]);
        const float y1 = x1 * cs - x2 * sn, y2 = x2 * cs + x1 * sn;
        if (head < H) {
            T* qd = q_out + static_cast<size_t>(r) * H * hd + head * hd;
            qd[d] = fromf<T>(y1);
            qd[d + half] = fromf<T>(y2);
        } else {
            const size_t base = kv_index<T>(kv, layer, s, p, head - H);
            kc[base + d] = fromf<T>(y1);
            kc[base + d + half] = fromf<T>(y2);
        }
    }
    for (int i = threadIdx.x; i < KV * hd; i += blockDim.x) {
        const int h = i / hd, d = i % hd;
        vc[kv_index<T>(kv, layer, s, p, h) + d] = src[(H + KV) * hd + i];
    }
}

// ------------------------------------------------ decode attention (GQA)
// One CTA per (row, kv head, split).  Lanes are grouped LPP per position;
// each lane holds VEC contiguous head dims of K/V (16-byte loads) and the G
// query heads of its kv group, with a per-group online softmax.
template <class T, int HD, int G>
__global__ void __launch_bounds__(128)
    attn_decode(const T* __restrict__ q, T* out, KvView kv, int layer,
                const int32_t* __restrict__ slot, const int32_t* __restrict__ pos, int rows,
                int split_len, float* ws_o, float* ws_ml) {
    pdl_trigger();
    pdl_wait();
    constexpr int VEC = 16 / sizeof(T);
    constexpr int LPP = HD / VEC;
    static_assert(LPP >= 1 && LPP <= 32 && (32 % LPP) == 0, "head dim / vector mismatch");
    constexpr int PPW = 32 / LPP;
    const int r = blockIdx.x, h = blockIdx.y, sp = blockIdx.z, nsp = gridDim.z;
    if (r >= rows) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / LPP, sub = lane % LPP;
    const int ctx = pos[r] + 1, s = slot[r];
    const int slen = split_len > 0 ? split_len : (ctx + nsp - 1) / nsp;  // per-row split (graphs)
    const int p0 = sp * slen, p1 = min(ctx, p0 + slen);
    const int H = kv.kv_heads * G;
    const float scale = rsqrtf(static_cast<float>(HD));

    float qv[G][VEC];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const T* qr = q + static_cast<size_t>(r) * H * HD + (h * G + g) * HD + sub * VEC;
#pragma unroll
        for (int e = 0; e < VEC; ++e) qv[g][e] = tof(qr[e]) * scale;
    }
    float m[G], l[G], acc[G][VEC];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        m[g] = -INFINITY;
        l[g] = 0.0f;
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[g][e] = 0.0f;
    }
    const T* kc = static_cast<const T*>(kv.k);
    const T* vc = static_cast<const T*>(kv.v);
    // U positions per lane group per iteration: all K/V loads are issued
    // before any math so each lane keeps 2U 16-byte loads in flight.
    constexpr int U = 4;
    for (int pb = p0 + warp * PPW * U; pb < p1; pb += 4 * PPW * U) {  // warp-uniform trip count
        uint4 kr[U], vr[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int p = pb + u * PPW + grp;
            if (p < p1) {
                const size_t base = kv_index<T>(kv, layer, s, p, h) + sub * VEC;
                kr[u] = __ldg(reinterpret_cast<const uint4*>(kc + base));
                vr[u] = __ldg(reinterpret_cast<const uint4*>(vc + base));
            } else {
                kr[u] = make_uint4(0, 0, 0, 0);
                vr[u] = make_uint4(0, 0, 0, 0);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool valid = pb + u * PPW + grp < p1;
            const T* kk = reinterpret_cast<const T*>(&kr[u]);
            const T* vv = reinterpret_cast<const T*>(&vr[u]);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                float sc = 0.0f;
#pragma unroll
                for (int e = 0; e < VEC; ++e) sc = fmaf(qv[g][e], tof(kk[e]), sc);
#pragma unroll
                for (int o = LPP / 2; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
                if (valid) {
                    const float mn = fmaxf(m[g], sc);
                    const float corr = __expf(m[g] - mn), pe = __expf(sc - mn);
                    l[g] = l[g] * corr + pe;
#pragma unroll
                    for (int e = 0; e < VEC; ++e) acc[g][e] = fmaf(acc[g][e], corr, pe * tof(vv[e]));
                    m[g] = mn;
                }
            }
        }
    }
    // combine the 4*PPW position groups of the CTA
    __shared__ float sm_ml[4 * PPW][G][2];
    __shared__ float sm_acc[4 * PPW][G][HD];
    const int gi = warp * PPW + grp;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        if (sub == 0) {
            sm_ml[gi][g][0] = m[g];
            sm_ml[gi][g][1] = l[g];
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) sm_acc[gi][g][sub * VEC + e] = acc[g][e];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
        const int g = i / HD, d = i % HD;
        float mx = -INFINITY;
        for (int j = 0; j < 4 * PPW; ++j) mx = fmaxf(mx, sm_ml[j][g][0]);
        float lsum = 0.0f, a = 0.0f;
        if (mx > -INFINITY) {
            for (int j = 0; j < 4 * PPW; ++j) {
                const float c = __expf(sm_ml[j][g][0] - mx);
                lsum += sm_ml[j][g][1] * c;
                a += sm_acc[j][g][d] * c;
            }
        }
        const int head = h * G + g;
        if (nsp == 1) {
            out[static_cast<size_t>(r) * H * HD + head * HD + d] = fromf<T>(lsum > 0.f ? a / lsum : 0.f);
        } else {
            const size_t o = (static_cast<size_t>(r) * H + head) * nsp + sp;
            ws_o[o * HD + d] = a;
            if (d == 0) {
                ws_ml[o * 2] = mx;
                ws_ml[o * 2 + 1] = lsum;
            }
        }
    }
}

template <class T>
__global__ void attn_split_combine(const float* ws_o, const float* ws_ml, T* out, int rows,
                                   int H, int hd, int nsp) {
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x, head = blockIdx.y;
    if (r >= rows) return;
    const size_t o = (static_cast<size_t>(r) * H + head) * nsp;
    float mx = -INFINITY;
    for (int j = 0; j < nsp; ++j) mx = fmaxf(mx, ws_ml[(o + j) * 2]);
    for (int d = threadIdx.x; d < hd; d += blockDim.x) {
        float l = 0.f, a = 0.f;
        if (mx > -INFINITY)
            for (int j = 0; j < nsp; ++j) {
                const float mj = ws_ml[(o + j) * 2];
                if (mj == -INFINITY) continue;
                const float c = __expf(mj - mx);
                l += ws_ml[(o + j) * 2 + 1] * c;
                a += ws_o[(o + j) * hd + d] * c;
            }
        out[(static_cast<size_t>(r) * H + head) * hd + d] = fromf<T>(l > 0.f ? a / l : 0.f);
    }
}

// ------------------------------------------------ prefill attention (GQA)
// One CTA per (query block of <= 32 consecutive rows of one slot, q head):
// 4 threads per query, each owning HD/4 dims; K/V tiles of 64 positions are
// staged in shared memory and reused by the block's 32 queries.
struct QBlock {
    int32_t row0;   // first row of the block
    int32_t n;      // rows (<= 32)
    int32_t slot;
    int32_t pos0;   // cache position of row0 (rows are consecutive positions)
};

template <class T, int HD>
__global__ void __launch_bounds__(128)
    attn_prefill(const T* __restrict__ q, T* out, KvView kv, int layer,
                 const QBlock* __restrict__ blocks, int n_heads) {
    pdl_trigger();
    pdl_wait();
    constexpr int TILE = HD >= 128 ? 32 : 64, DPT = HD / 4;  // <= 48 KB static smem
    const QBlock b = blocks[blockIdx.x];
    const int head = blockIdx.y, G = n_heads / kv.kv_heads, h = head / G;
    const int qi = threadIdx.x >> 2, part = threadIdx.x & 3;
    const bool active = qi < b.n;
    const int qpos = b.pos0 + qi;
    const float scale = rsqrtf(static_cast<float>(HD));
    __shared__ float sk[TILE][HD + 1];
    __shared__ float sv[TILE][HD + 1];
    float qv[DPT], acc[DPT];
    const T* qr = q + (static_cast<size_t>(b.row0 + (active ? qi : 0)) * n_heads + head) * HD +
                  part * DPT;
#pragma unroll
    for (int e = 0; e < DPT; ++e) {
        qv[e] = tof(qr[e]) * scale;
        acc[e] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    const int last = b.pos0 + b.n - 1;
    const T* kc = static_cast<const T*>(kv.k);
    const T* vc = static_cast<const T*>(kv.v);
    for (int t0 = 0; t0 <= last; t0 += TILE) {
        const int tn = min(TILE, last + 1 - t0);
        for (int i = threadIdx.x; i < tn * HD; i += blockDim.x) {
            const int p = i / HD, d = i % HD;
            const size_t idx = kv_index<T>(kv, layer, b.slot, t0 + p, h) + d;
            sk[p][d] = tof(kc[idx]);
            sv[p][d] = tof(vc[idx]);
        }
        __syncthreads();
        for (int p = 0; p < tn; ++p) {  // uniform trip count; causal mask below
            float sc = 0.f;
#pragma unroll
            for (int e = 0; e < DPT; ++e) sc = fmaf(qv[e], sk[p][part * DPT + e], sc);
            sc += __shfl_xor_sync(0xffffffffu, sc, 1);
            sc += __shfl_xor_sync(0xffffffffu, sc, 2);
            if (t0 + p <= qpos) {
                const float mn = fmaxf(m, sc);
                const float corr = __expf(m - mn), pe = __expf(sc - mn);
                l = l * corr + pe;
#pragma unroll
                for (int e = 0; e < DPT; ++e) acc[e] = fmaf(acc[e], corr, pe * sv[p][part * DPT + e]);
                m = mn;
            }
        }
        __syncthreads();
    }
    if (active) {
        T* o = out + (static_cast<size_t>(b.row0 + qi) * n_heads + head) * HD + part * DPT;
#pragma unroll
        for (int e = 0; e < DPT; ++e) o[e] = fromf<T>(l > 0.f ? acc[e] / l : 0.f);
    }
}

// ---------------------------------------------- sampling / log-prob combine
// Reduces the lm_head GEMM's per-block partials of one row (one warp per row):
// log-sum-exp over the vocabulary, then either
//   sampling: block b* = argmax_b (lse_b + Gumbel(key ^ kBlockKey, b)) (ties to
//     the lower block), token = the block's inverse-CDF pick, log-prob =
//     its logit - lse; or
//   scoring: log-prob of the given target = target logit - lse.
static __global__ void logits_combine(const float4* __restrict__ partials, int n_tiles, int vocab,
                                      int rows, const uint64_t* keys, const float* tgt_logit,
                                      const int32_t* __restrict__ slot,
                                      const int32_t* __restrict__ tidx, int32_t* tok_buf,
                                      float* lp_buf, int buf_stride, float* lse_out,
                                      int32_t* tok_rows, int32_t* iter_inc = nullptr) {
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (iter_inc && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(iter_inc, 1);  // next decode step
    if (r >= rows) return;
    const float4* pr = partials + static_cast<size_t>(r) * n_tiles;
    float mx = -INFINITY;
    for (int i = lane; i < n_tiles; i += 32) mx = fmaxf(mx, pr[i].x);
    mx = warp_max(mx);
    float s = 0.f, best = -INFINITY;
    int bb = 0x7fffffff;
    const uint64_t bkey = keys ? keys[r] ^ kBlockKey : 0;
    for (int i = lane; i < n_tiles; i += 32) {
        const float4 v = pr[i];
        if (v.x > -INFINITY) s += v.y * __expf(v.x - mx);
        if (keys) {
            const float sc = v.x + logf(v.y) + gumbel_noise(bkey, static_cast<uint32_t>(i));
            if (sc > best || (sc == best && i < bb)) {
                best = sc;
                bb = i;
            }
        }
    }
    s = warp_sum(s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float b2 = __shfl_xor_sync(0xffffffffu, best, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bb, o);
        if (b2 > best || (b2 == best && i2 < bb)) {
            best = b2;
            bb = i2;
        }
    }
    if (lane != 0) return;
    const float lse = mx + logf(s);
    if (lse_out) lse_out[r] = lse;
    const size_t at = slot ? static_cast<size_t>(slot[r]) * buf_stride + tidx[r] : r;
    if (keys) {
        if (bb < 0 || bb >= n_tiles) bb = 0;  // memory safety only (non-finite logits)
        const float4 v = pr[bb];
        int tok = __float_as_int(v.z);
        if (tok < 0 || tok >= vocab) tok = 0;
        tok_buf[at] = tok;
        lp_buf[at] = v.w - lse;
        if (tok_rows) tok_rows[r] = tok;
    } else if (lp_buf) {
        lp_buf[at] = tgt_logit[r] - lse;
    }
}

// -------------------------------------------------------- row construction
struct DecodeSeq {   // per decode row (sorted by remaining length, descending)
    int32_t slot;
    int32_t prompt_len;
    int32_t generated;  // g at step start
    int32_t target_len;
    int64_t id;
};

// Rows of decode iteration `it` (1-based): row r produces response token
// j = g + it from input token j-1 (or the last prompt token) at position P+j-2.
static __global__ void decode_rows(const DecodeSeq* __restrict__ seqs, int rows,
                                   const int32_t* __restrict__ iter,
                                   const int32_t* __restrict__ prompt_buf, int prompt_stride,
                                   const int32_t* __restrict__ tok_buf, int tok_stride,
                                   uint64_t seed, RowMeta meta, int dummy_slot) {
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int it = *iter;  // device-resident so one captured graph serves every iteration
    DecodeSeq s = seqs[r];
    if (s.generated + it > s.target_len) {  // finished (or padding) row of a bucketed batch:
        s.slot = dummy_slot;                 // decode into the scratch slot instead
        s.prompt_len = 1;
        s.generated = 0;
        s.id = -1;
    }
    const int j = s.generated + it;
    meta.slot[r] = s.slot;
    meta.pos[r] = s.prompt_len + j - 2;
    meta.tok[r] = j == 1 ? prompt_buf[s.slot * prompt_stride + s.prompt_len - 1]
                         : tok_buf[s.slot * tok_stride + j - 1];
    meta.t[r] = j;
    meta.key[r] = token_key(seed, s.id, j);
}

struct Segment {     // a run of consecutive cache positions of one slot
    int32_t slot;
    int32_t pos0;
    int32_t n;
    int32_t row0;
    int32_t prompt_len;
    int32_t _pad;
};

// Expands segments into rows (one CTA per segment).  Token at position q:
// prompt[q] for q < P, else response token q-P+1.
static __global__ void segment_rows(const Segment* __restrict__ segs, const int32_t* __restrict__ prompt_buf,
                             int prompt_stride, const int32_t* __restrict__ tok_buf, int tok_stride,
                             RowMeta meta) {
    const Segment s = segs[blockIdx.x];
    for (int i = threadIdx.x; i < s.n; i += blockDim.x) {
        const int q = s.pos0 + i, r = s.row0 + i;
        meta.slot[r] = s.slot;
        meta.pos[r] = q;
        meta.tok[r] = q < s.prompt_len ? prompt_buf[s.slot * prompt_stride + q]
                                       : tok_buf[s.slot * tok_stride + q - s.prompt_len + 1];
        meta.t[r] = q - s.prompt_len + 2;
    }
}

// Scatter a per-row head output to [slot][t] (t in [t_lo, t_hi]).
static __global__ void scatter_rows(const float* __restrict__ v, const int32_t* __restrict__ slot,
                             const int32_t* __restrict__ tidx, int rows, float* buf, int stride,
                             int t_lo, const int32_t* __restrict__ t_hi_per_slot, int t_hi_offset) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int t = tidx[r], s = slot[r];
    const int hi = t_hi_per_slot[s] + t_hi_offset;
    if (t >= t_lo && t <= hi) buf[static_cast<size_t>(s) * stride + t] = v[r];
}

// Reward: row whose output index is L+1 (the last response token).
static __global__ void reward_rows(const float* __restrict__ v, const int32_t* __restrict__ slot,
                            const int32_t* __restrict__ tidx, int rows,
                            const int32_t* __restrict__ target_len, float* reward) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int s = slot[r];
    if (tidx[r] == target_len[s] + 1) reward[s] = v[r];
}

// Reference-model lm_head rows: gather hidden rows (from this wave's hidden
// buffer or the per-slot pending buffer) with their target tokens.
struct LmRow {
    int32_t src;     // >= 0: row of the wave hidden buffer; < 0: -(slot+1) pending row
    int32_t slot;
    int32_t t;       // response index of the target
    int32_t _pad;
};
template <class T>
__global__ void gather_lm_rows(const LmRow* __restrict__ rows, int n, const T* __restrict__ hid,
                               const T* __restrict__ pending, int d,
                               const int32_t* __restrict__ tok_buf, int tok_stride, T* out,
                               int32_t* tgt, int32_t* slot_out, int32_t* t_out) {
    const int r = blockIdx.x;
    if (r >= n) return;
    const LmRow lr = rows[r];
    const T* src = lr.src >= 0 ? hid + static_cast<size_t>(lr.src) * d
                               : pending + static_cast<size_t>(-lr.src - 1) * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) out[static_cast<size_t>(r) * d + i] = src[i];
    if (threadIdx.x == 0) {
        tgt[r] = tok_buf[lr.slot * tok_stride + lr.t];
        slot_out[r] = lr.slot;
        t_out[r] = lr.t;
    }
}
template <class T>
__global__ void store_pending(const int32_t* __restrict__ src_rows, const int32_t* __restrict__ slots,
                              int n, const T* __restrict__ hid, T* pending, int d) {
    const int r = blockIdx.x;
    if (r >= n) return;
    const T* s = hid + static_cast<size_t>(src_rows[r]) * d;
    T* dst = pending + static_cast<size_t>(slots[r]) * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = s[i];
}

static __global__ void set_int(int32_t* p, int v) { *p = v; }

// Synthetic prompt tokens keyed by (seed, sequence id, position).
static __global__ void prompt_tokens(int32_t* prompt_buf, int stride, const int32_t* slots,
                              const int64_t* ids, const int32_t* lens, int n, uint64_t seed,
                              int vocab) {
    const int i = blockIdx.x;
    if (i >= n) return;
    for (int q = threadIdx.x; q < lens[i]; q += blockDim.x) {
        const uint64_t h = mix64(seed ^ 0x70726f6d7074ull ^ mix64(static_cast<uint64_t>(ids[i]) * 0x100000001b3ull + q));
        prompt_buf[slots[i] * stride + q] = static_cast<int32_t>(h % static_cast<uint64_t>(vocab));
    }
}

}  // namespace oppo
