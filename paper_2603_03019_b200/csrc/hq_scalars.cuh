// hq_scalars.cuh -- the per-layer scalar step shared by k_scalars2 (hq_v2.cu) and the
// fused tail of the sweep kernel (hq_v3.cu).  Product code only.
//
// Given the per-layer sums S[n][v] of one half-sweep (v: V2_P, V2_OM, V2_KA, V2_LAM,
// V2_DL1) or of the init / residual passes, update the scalar block `sb` (a shared-memory
// copy of the V2S_* block):
//   lambda(n) (Eq. lambdaHeter), mu(n) (Eq. muHeter via the exact flow
//   identity sum_m p den = mu* + lambda_old(n)), the a-priori
//   normalisers alpha(n) = mu*(n)/lambda(n-1) and beta(n) = lambda(n)/mu(n+1) of the next
//   half-sweep, and p(n) by Eq. bnd_stationary.
// Called by every thread of the block (contains __syncthreads); layers are processed in
// parallel, the prefix product of Eq. bnd_stationary and the proxy sum by thread 0, so the
// result does not depend on the block size.
#pragma once
#include "hq_internal.h"
#include "hq_v2.h"

// Per-layer sums of the transposed CTA partials partial[(L * HQ_NV + v) * G + cta] of a
// sweep launch, layers 0..N: a group of tpi = 2^lg threads per (layer, value) (lg 0..5),
// each thread with four interleaved accumulators (loads in flight), combined in a fixed
// order (deterministic).  No barrier.
// only: 0 = every layer 0..N, else a mask of the layers to reduce (the others are left as they are)
__device__ __forceinline__ void reduce_partials_t(const double *partial, int G, int N, double (*S)[NV2], int lg,
                                                  uint32_t only = 0u) {
    int lay[HQ_NL];   // the reduced layers, ascending
    int nl = 0;
    for (int L = 0; L <= N; L++)
        if (!only || ((only >> L) & 1u)) lay[nl++] = L;
    const int items = nl * NV2;
    const int tpi = 1 << lg, q = threadIdx.x & (tpi - 1);
    // items rounded up to whole warps: every warp visits its items together, so the
    // shuffles below are warp-uniform (blockDim.x is a multiple of 32)
    const int per_warp = 32 >> lg;
    const int nit = (items + per_warp - 1) / per_warp * per_warp;
    for (int it = threadIdx.x >> lg; it < nit; it += blockDim.x >> lg) {
        const int li = it / NV2, v = it - li * NV2;
        const bool ok = li < nl;
        const int L = ok ? lay[li] : 0;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (ok) {
            const double *src = partial + ((size_t)L * HQ_NV + v) * G;
            int b = q;
            for (; b + 3 * tpi < G; b += 4 * tpi) {
                s0 += src[b];
                s1 += src[b + tpi];
                s2 += src[b + 2 * tpi];
                s3 += src[b + 3 * tpi];
            }
            for (; b < G; b += tpi) s0 += src[b];
        }
        double s = (s0 + s1) + (s2 + s3);
        for (int o = 1; o < tpi; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (q == 0 && ok) S[L][v] = s;
    }
}

// The same reduction read through L2 (k_loop3: the partials were written by other CTAs in
// the same kernel, an SM may hold stale L1 lines of the buffer from two phases earlier).
__device__ __forceinline__ void reduce_partials_t_cg(const double *partial, int G, int N, double (*S)[NV2], int lg,
                                                  uint32_t only = 0u) {
    int lay[HQ_NL];   // the reduced layers, ascending
    int nl = 0;
    for (int L = 0; L <= N; L++)
        if (!only || ((only >> L) & 1u)) lay[nl++] = L;
    const int items = nl * NV2;
    const int tpi = 1 << lg, q = threadIdx.x & (tpi - 1);
    // items rounded up to whole warps: every warp visits its items together, so the
    // shuffles below are warp-uniform (blockDim.x is a multiple of 32)
    const int per_warp = 32 >> lg;
    const int nit = (items + per_warp - 1) / per_warp * per_warp;
    for (int it = threadIdx.x >> lg; it < nit; it += blockDim.x >> lg) {
        const int li = it / NV2, v = it - li * NV2;
        const bool ok = li < nl;
        const int L = ok ? lay[li] : 0;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (ok) {
            const double *src = partial + ((size_t)L * HQ_NV + v) * G;
            int b = q;
            for (; b + 3 * tpi < G; b += 4 * tpi) {
                s0 += __ldcg(src + b);
                s1 += __ldcg(src + b + tpi);
                s2 += __ldcg(src + b + 2 * tpi);
                s3 += __ldcg(src + b + 3 * tpi);
            }
            for (; b < G; b += tpi) s0 += __ldcg(src + b);
        }
        double s = (s0 + s1) + (s2 + s3);
        for (int o = 1; o < tpi; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (q == 0 && ok) S[L][v] = s;
    }
}

__device__ __forceinline__ void scalars_update(int N, int full_lists, double Lam, int mode, int c, uint32_t active,
                                               const double (*S)[NV2], double *sb) {
    double *lam = sb + V2S_LAM, *mu = sb + V2S_MU, *al = sb + V2S_ALPHA, *be = sb + V2S_BETA;
    double *pn1 = sb + V2S_PN, *om = sb + V2S_OM, *ka = sb + V2S_KA, *misc = sb + V2S_MISC;
    const int tid = threadIdx.x;
    __shared__ double s_g[HQ_NL];
    __shared__ double s_tot;
    __shared__ int s_err;
    if (tid == 0) s_err = 0;
    if (mode == 2) {
        if (tid == 0) {
            double num = 0.0, den = 0.0;
            for (int L = 0; L <= N; L++) {
                sb[V2S_RNUM + L] = S[L][V2_RNUM];
                sb[V2S_RDEN + L] = S[L][V2_RDEN];
                num += S[L][V2_RNUM];
                den += S[L][V2_RDEN];
            }
            misc[1] = num / den;
        }
        __syncthreads();
        return;
    }
    __syncthreads();
    if (mode == 0) {
        // init: S = {sum p, sum p mu_m, sum p omega, sum p kappa, sum p lambda_m} over both classes
        for (int L = tid; L <= N; L += blockDim.x) {
            lam[L] = S[L][4];
            mu[L] = S[L][1];
            om[L] = S[L][2];
            ka[L] = S[L][3];
            sb[V2S_SUMP + L] = S[L][0];
            sb[V2S_DL1 + L] = 0.0;
        }
        c = 0;   // the first half-sweep updates class 1
    } else {
        // layers of one parity: lambda(L-1) of the other parity is read, never written here
        for (int L = 1 + tid; L <= N - 1; L += blockDim.x) {
            if (!((active >> L) & 1u)) continue;
            const double lnew = full_lists ? Lam * S[L][V2_P] : S[L][V2_LAM];
            const double mstar = al[L] * lam[L - 1];
            const double mnew = mstar + lam[L] - lnew;
            sb[V2S_MUSTAR + L] = mstar;
            lam[L] = lnew;
            mu[L] = mnew;
            om[L] = S[L][V2_OM];
            ka[L] = S[L][V2_KA];
            sb[V2S_SUMP + L] = S[L][V2_P];
            sb[V2S_DL1 + L] = S[L][V2_DL1];
            if (!(S[L][V2_P] > 0.0) || !isfinite(mnew)) s_err = 1;
        }
    }
    __syncthreads();
    // coefficients for the next half-sweep (class 1 - c)
    const int nc = 1 - c;
    for (int L = 1 + tid; L <= N - 1; L += blockDim.x) {
        if ((L & 1) != nc) continue;
        const double b = lam[L] / mu[L + 1];
        const double a = (1.0 - b * ka[L + 1]) / om[L - 1];
        be[L] = b;
        al[L] = a;
        if (!(om[L - 1] > 0.0) || !isfinite(a) || !(a > 0.0)) s_err = 1;
    }
    // Eq. bnd_stationary: ratios in parallel, prefix product by thread 0
    for (int L = 1 + tid; L <= N; L += blockDim.x) s_g[L] = lam[L - 1] / mu[L];
    __syncthreads();
    if (tid == 0) {
        double prod = 1.0, tot = 1.0;
        s_g[0] = 1.0;
        for (int L = 1; L <= N; L++) {
            prod *= s_g[L];
            s_g[L] = prod;
            tot += prod;
        }
        s_tot = tot;
    }
    __syncthreads();
    for (int L = tid; L < 34; L += blockDim.x) pn1[L] = (L >= 1 && L <= N + 1) ? s_g[L - 1] / s_tot : 0.0;
    __syncthreads();
    if (tid == 0) {
        double prox = 0.0;
        for (int L = 1; L <= N - 1; L++) prox += pn1[L + 1] * sb[V2S_DL1 + L];
        misc[2] = prox;
        if (s_err) misc[0] = 1.0;
    }
    __syncthreads();
}
