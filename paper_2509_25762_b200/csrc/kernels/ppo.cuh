// ppo.cuh — fused per-token PPO kernels (K7-K10, K12).
//
// Ragged batch layout: n_seq sequences, offsets[n_seq+1] token prefix sums;
// per-token arrays indexed by offsets[i]+t (t = 0..len-1); values hold len+1
// entries per sequence at offsets[i]+i (terminal value included).
// Reference semantics: compute_gae / terminal_rewards (ppo.cpp:71-91),
// clipped_objective (ppo.cpp:101-120), clipped_objective_grad's per-token
// scalar (ppo.cpp:138-177), tabular value fit (ppo.cpp:292-315).
#pragma once

#include "common.cuh"

namespace oppo {

template <class R> __device__ __forceinline__ R mul_rn(R a, R b);
template <> __device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
template <class R> __device__ __forceinline__ R add_rn(R a, R b);
template <> __device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

// Per-token reward: -kl_coef * (old_lp - ref_lp) (k1 estimator of KL(pi_old || pi_ref)),
// plus the sequence score on the last token (terminal_rewards, ppo.cpp:87-91).
template <class R>
__global__ void token_rewards(int n_seq, const int32_t* __restrict__ off, const R* __restrict__ score,
                              const R* __restrict__ old_lp, const R* __restrict__ ref_lp, R kl_coef,
                              R* __restrict__ rew, R* __restrict__ kl) {
    const int i = blockIdx.x;
    if (i >= n_seq) return;
    const int a = off[i], b = off[i + 1];
    for (int t = a + threadIdx.x; t < b; t += blockDim.x) {
        R k = 0;
        if (ref_lp) k = old_lp[t] - ref_lp[t];
        if (kl) kl[t] = k;
        R r = kl_coef != R(0) ? -kl_coef * k : R(0);
        if (t == b - 1) r = add_rn(r, score[i]);
        rew[t] = r;
    }
}

// GAE reverse recursion (compute_gae, ppo.cpp:71-85), one warp per sequence.
// Each lane owns a contiguous chunk of the sequence.
//   fp64 (parity): lanes run right-to-left one after another, handing the
//     running advantage over by shuffle, so every add/multiply happens in the
//     reference's order (bit-identical to compute_gae).
//   fp32 (production): each lane folds its chunk into an affine map
//     A_start = L + c^n A_end (c = gamma*lambda); a log-step suffix scan over
//     lanes composes the maps, then each lane replays its chunk from the carry.
// returns = adv + V.
template <class R>
__global__ void gae_scan(int n_seq, const int32_t* __restrict__ off, const R* __restrict__ rew,
                         const R* __restrict__ values, R gamma, R lambda, R* __restrict__ adv,
                         R* __restrict__ ret) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= n_seq) return;
    const int a = off[warp], len = off[warp + 1] - a;
    const R* v = values + a + warp;  // len+1 values
    const R c = mul_rn(gamma, lambda);
    const int per = (len + 31) / 32;
    const int s = min(len, lane * per), e = min(len, s + per);
    auto delta = [&](int t) {  // r_t + gamma*V_{t+1} - V_t, no FMA contraction
        return add_rn(add_rn(rew[a + t], mul_rn(gamma, v[t + 1])), -v[t]);
    };
    R run = 0;
    if constexpr (sizeof(R) == 8) {
        for (int k = 31; k >= 0; --k) {
            if (lane == k)
                for (int t = e - 1; t >= s; --t) {
                    run = add_rn(delta(t), mul_rn(c, run));
                    adv[a + t] = run;
                    ret[a + t] = add_rn(run, v[t]);
                }
            run = __shfl_sync(0xffffffffu, run, k);
        }
    } else {
        R l = 0, cp = 1;
        for (int t = e - 1; t >= s; --t) {
            l = delta(t) + c * l;
            cp *= c;
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {  // suffix composition of lane maps
            const R l2 = __shfl_down_sync(0xffffffffu, l, o);
            const R c2 = __shfl_down_sync(0xffffffffu, cp, o);
            if (lane + o < 32) {
                l = l + cp * l2;
                cp = cp * c2;
            }
        }
        R carry = __shfl_down_sync(0xffffffffu, l, 1);  // A at the start of lane+1's chunk
        if (lane == 31) carry = 0;
        run = carry;
        for (int t = e - 1; t >= s; --t) {
            run = delta(t) + c * run;
            adv[a + t] = run;
            ret[a + t] = run + v[t];
        }
    }
}

// Critic target of the reference's value fit (ppo.cpp:296-314): the
// gamma-discounted return of terminal_rewards, ret_t = gamma^(L-1-t) * score,
// accumulated in the reference's order (ret = r_t + gamma * ret, right to left).
template <class R>
__global__ void mc_returns(int n_seq, const int32_t* __restrict__ off, const R* __restrict__ score, R gamma,
                           R* __restrict__ ret) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_seq) return;
    const int a = off[i], len = off[i + 1] - a;
    R run = 0;
    for (int t = len - 1; t >= 0; --t) {
        run = add_rn(t == len - 1 ? score[i] : R(0), mul_rn(gamma, run));
        ret[a + t] = run;
    }
}

// Block-partial sums for whitening statistics: [sum adv, sum adv^2, count].
template <class R>
__global__ void moments(const R* __restrict__ x, int n, double* __restrict__ partial) {
    double s = 0, s2 = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double v = static_cast<double>(x[i]);
        s += v;
        s2 += v * v;
    }
    s = warp_sum_d(s);
    s2 = warp_sum_d(s2);
    __shared__ double sh[2][32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sh[0][w] = s;
        sh[1][w] = s2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int i = 0; i < (blockDim.x >> 5); ++i) {
            a += sh[0][i];
            b += sh[1][i];
        }
        partial[blockIdx.x * 2] = a;
        partial[blockIdx.x * 2 + 1] = b;
    }
}
static __global__ void moments_final(const double* __restrict__ partial, int nblk, double n, double* out) {
    if (threadIdx.x != 0) return;
    out[2] = n;
    double a = 0, b = 0;
    for (int i = 0; i < nblk; ++i) {  // fixed order: deterministic
        a += partial[i * 2];
        b += partial[i * 2 + 1];
    }
    out[0] = a;
    out[1] = b;
}

// Clipped surrogate per token (+ optional whitening with global stats):
//   r = exp(new - old); obj_t = min(r A, clip(r, 1-eps, 1+eps) A)
//   dobj/dlogp_t = (1/N) * dterm * r, dterm from the branch rule of
//   clipped_objective_grad (ppo.cpp:163-168).
// Writes per-token dobj/dlogp and per-block partial sums of obj_t.
template <class R>
__global__ void ppo_clip(int n, const R* __restrict__ new_lp, const R* __restrict__ old_lp,
                         R* __restrict__ adv, R eps, const double* stats /* sum,sumsq,n or null */,
                         double whiten_eps, R* __restrict__ dobj, double* __restrict__ obj_partial,
                         R inv_n) {
    double acc = 0;
    R mean = 0, rstd = 1;
    if (stats) {
        const double cnt = stats[2];
        const double mu = stats[0] / cnt;
        const double var = stats[1] / cnt - mu * mu;
        mean = static_cast<R>(mu);
        rstd = static_cast<R>(1.0 / sqrt(fmax(var, 0.0) + whiten_eps));
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        R a = adv[i];
        if (stats) {
            a = (a - mean) * rstd;
            adv[i] = a;
        }
        const R ratio = exp(new_lp[i] - old_lp[i]);
        const R unclipped = ratio * a;
        const R cl = ratio < R(1) - eps ? R(1) - eps : (ratio > R(1) + eps ? R(1) + eps : ratio);
        const R clipped = cl * a;
        acc += static_cast<double>(unclipped < clipped ? unclipped : clipped);
        R dterm;
        if (unclipped <= clipped) dterm = a;
        else dterm = (ratio > R(1) - eps && ratio < R(1) + eps) ? a : R(0);
        dobj[i] = inv_n * dterm * ratio;
    }
    acc = warp_sum_d(acc);
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0;
        for (int i = 0; i < (blockDim.x >> 5); ++i) s += sh[i];
        obj_partial[blockIdx.x] = s;
    }
}

// out[0] += sum of block partials (fixed order): accumulates the clipped
// objective over the micro-batches of the full-parameter update.
static __global__ void sum_partials_acc(const double* p, int n, double* out) {
    if (threadIdx.x) return;
    double s = 0;
    for (int i = 0; i < n; ++i) s += p[i];
    out[0] += s;
}

// Value-head regression on the critic's cached hidden states:
// grad_w = (1/N) sum_t (V_t - R_t) h_t ; loss = (1/2N) sum_t (V_t - R_t)^2.
// One CTA per 64-column slab of w, deterministic order over tokens.
template <class T>
__global__ void value_head_grad(const T* __restrict__ hid, int d, int n,
                                const float* __restrict__ v, const float* __restrict__ target,
                                float* __restrict__ grad, float inv_n) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= d) return;
    float g = 0.f;
    for (int t = 0; t < n; ++t) g = fmaf(v[t] - target[t], tof(hid[static_cast<size_t>(t) * d + col]), g);
    grad[col] = g * inv_n;
}

}  // namespace oppo
