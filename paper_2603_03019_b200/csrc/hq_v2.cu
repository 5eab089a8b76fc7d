// hq_v2.cu -- per-instance precompute and the per-half-sweep scalar step of the tiled path
// (N >= 9, hq_v3.cu), and the assembly of pi.
//
//  * k_lambda_states: lambda_m for truncated lists (Lambda minus the atoms whose whole list
//    is busy), per state.
//  * k_omkap: the scatter weights of the a-priori normalisation (R13)
//        omega(l) = sum_{i not in l} lambda_{l, l+i} / den(l+i),
//        kappa(l) = sum_{i in l}     nu_i              / den(l-i),
//    since sum_{m in C_n} a_m = sum_{l in C_{n-1}} p(l) omega(l) / lambda(n-1) and
//    sum_{m in C_n} b_m = lambda(n)/mu(n+1) sum_{l in C_{n+1}} p(l) kappa(l) (exact
//    re-indexing of the sums in Eq. updateHeter), so one pass per
//    half-sweep writes p_n(m) = (alpha_n A(m) + beta_n D(m)) / den(m) directly.
//  * k_scalars2: lambda(n), mu(n) (Eqs. lambdaHeter / muHeter), the normalisers
//    alpha(n) = mu*(n)/lambda(n-1), beta(n) = lambda(n)/mu(n+1) and p(n)
//    (Eq. bnd_stationary) from the fixed-order sums of the CTA partials.
//  * k_assemble2: pi(m) = p(n) p_n(m) scattered to the ABI unit order.
// (The round-1 warp-tiled sweep kernel for N = 8 was retired in round 2: N < 9 runs the
// two-pass kernels of hq_kernels.cu.)
#include <cuda_runtime.h>
#include <cub/cub.cuh>
#include <cstdint>
#include "hq_internal.h"
#include "hq_v2.h"
#include "hq_scalars.cuh"

namespace hq2 {

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// ---------------------------------------------------------------------------
// Precompute 1: lambda_m for truncated lists (temp array, compressed layout).
// ---------------------------------------------------------------------------
__global__ void k_lambda_states(P2Args a, double *__restrict__ lamarr) {
    const uint64_t half = 1ull << (a.N - 1);
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < 2 * half;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const int c = (int)(x >= half);
        const uint32_t j = (uint32_t)(x - (c ? half : 0));
        const int b0 = c ^ (__popc(j) & 1);
        const uint32_t m = (j << 1) | (uint32_t)b0;
        double blocked = 0.0;
        int v = 0;
        while (v < a.nnodes) {
            const int2 nd = __ldg(&a.node[v]);
            if ((m >> (nd.x & 0xff)) & 1u) {
                blocked += __ldg(&a.lam_end[v]);
                v++;
            } else {
                v = nd.y;
            }
        }
        lamarr[x] = a.Lam - blocked;
    }
}

// ---------------------------------------------------------------------------
// Precompute 2: scatter weights omega(l), kappa(l) for every state.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double lam_of(const P2Args &a, const double *lamarr, uint32_t m) {
    if (a.full_lists) return (m == (1u << a.N) - 1u) ? 0.0 : a.Lam;
    const uint64_t half = 1ull << (a.N - 1);
    const int c = __popc(m) & 1;
    return lamarr[(c ? half : 0) + (m >> 1)];
}

__global__ void k_omkap(P2Args a, const double *__restrict__ lamarr, double2 *__restrict__ omkap) {
    const uint64_t half = 1ull << (a.N - 1);
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < 2 * half;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const int c = (int)(x >= half);
        const uint32_t j = (uint32_t)(x - (c ? half : 0));
        const int b0 = c ^ (__popc(j) & 1);
        const uint32_t l = (j << 1) | (uint32_t)b0;
        double up[HQ_MAXN + 1];
        for (int u = 0; u <= HQ_MAXN; u++) up[u] = 0.0;
        // out-rates of l: every atom goes to its first free unit (frontier nodes)
        int v = 0;
        while (v < a.nnodes) {
            const int2 nd = __ldg(&a.node[v]);
            const int u = nd.x & 0xff;
            if ((l >> u) & 1u) {
                v++;
            } else {
                up[u] += __ldg(&a.lam_thr[v]);
                v = nd.y;
            }
        }
        double mul = 0.0;
        for (int u = 0; u < a.N; u++)
            if ((l >> u) & 1u) mul += a.nu[u];
        double om = 0.0, ka = 0.0;
        for (int u = 0; u < a.N; u++) {
            const uint32_t nb = l ^ (1u << u);
            if ((l >> u) & 1u) {
                const double den = lam_of(a, lamarr, nb) + (mul - a.nu[u]);
                ka += a.nu[u] / den;
            } else if (up[u] != 0.0) {
                const double den = lam_of(a, lamarr, nb) + (mul + a.nu[u]);
                om += up[u] / den;
            }
        }
        omkap[x] = make_double2(om, ka);
    }
}

// ---------------------------------------------------------------------------
// Layer scalars (one block, warp n reduces layer n over the CTA partials).
//   mode 0 (init), 1 (after a sweep half-sweep), 2 (after a residual pass).
// After modes 0/1 the coefficients alpha(n), beta(n) of the next half-sweep
// (class 1 - c) are prepared:
//   beta(n)  = lambda(n) / mu(n+1)
//   alpha(n) = mu*(n) / lambda(n-1) = (1 - beta(n) S_kappa(n+1)) / S_omega(n-1)
// and p(n) (Eq. bnd_stationary) is refreshed.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_scalars2(int N, int full_lists, double Lam, int mode, int c, uint32_t active,
                                                    int ncta, const double *__restrict__ partial,
                                                    const double *blk, double *blk_out, int transposed) {
    __shared__ double S[HQ_NL][NV2];
    __shared__ double sblk[V2S_TOTAL];
    const int lane = threadIdx.x & 31, n = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < V2S_TOTAL; i += blockDim.x) sblk[i] = blk[i];
    if (transposed) {   // partial[(layer * HQ_NV + v) * ncta + cta]
        reduce_partials_t(partial, ncta, N, S, 5, mode == 1 ? active : 0u);   // one warp per (layer, value)
    } else if (n <= N) {
        double s[NV2];
#pragma unroll
        for (int v = 0; v < NV2; v++) s[v] = 0.0;
        for (int i = lane; i < ncta; i += 32)
#pragma unroll
            for (int v = 0; v < NV2; v++) s[v] += partial[((size_t)i * HQ_NL + n) * HQ_NV + v];
#pragma unroll
        for (int v = 0; v < NV2; v++) {
            s[v] = warp_sum(s[v]);
            if (lane == 0) S[n][v] = s[v];
        }
    }
    __syncthreads();
    // the scalar step runs on a shared-memory copy of the block
    scalars_update(N, full_lists, Lam, mode, c, active, S, sblk);
    for (int i = threadIdx.x; i < V2S_TOTAL; i += blockDim.x) blk_out[i] = sblk[i];
}

// pi[m_abi] = p(w(m)) p_{w(m)}(m), internal index m -> ABI index via perm.
__global__ void k_assemble2(int N, const double *__restrict__ pw, const double *__restrict__ pn1, PermArg perm,
                            double *__restrict__ pi) {
    const uint64_t S = 1ull << N, half = S >> 1;
    for (uint64_t m = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; m < S; m += (uint64_t)gridDim.x * blockDim.x) {
        const int n = __popcll(m);
        const uint64_t off = (n & 1) ? half : 0;
        uint64_t ma = 0;
        for (int u = 0; u < N; u++) ma |= ((m >> u) & 1ull) << perm.p[u];
        pi[ma] = pn1[n + 1] * pw[off + (m >> 1)];
    }
}

}  // namespace hq2

// ---------------------------------------------------------------------------
namespace hq2_launch {

int sweep_grid(int nsm) { return nsm * 2; }


cudaError_t lambda_states(const P2Args &a, double *lamarr, int grid, cudaStream_t s) {
    hq2::k_lambda_states<<<grid, 256, 0, s>>>(a, lamarr);
    return cudaGetLastError();
}
cudaError_t omkap(const P2Args &a, const double *lamarr, double2 *ok, int grid, cudaStream_t s) {
    hq2::k_omkap<<<grid, 256, 0, s>>>(a, lamarr, ok);
    return cudaGetLastError();
}
cudaError_t prog_scan(const uint32_t *size16, uint32_t *off16, uint64_t n, void *tmp, size_t *tmp_bytes,
                      cudaStream_t s) {
    return cub::DeviceScan::ExclusiveSum(tmp, *tmp_bytes, size16, off16, (int)n, s);
}
cudaError_t prog_max(const uint32_t *size16, uint32_t *out, uint64_t n, void *tmp, size_t *tmp_bytes, cudaStream_t s) {
    return cub::DeviceReduce::Max(tmp, *tmp_bytes, size16, out, (int)n, s);
}
cudaError_t scalars(int N, int full_lists, double Lam, int mode, int c, uint32_t active, int ncta,
                    const double *partial, double *blk, cudaStream_t s, int transposed, double *blk_out) {
    hq2::k_scalars2<<<1, 1024, 0, s>>>(N, full_lists, Lam, mode, c, active, ncta, partial, blk,
                                       blk_out ? blk_out : blk, transposed);
    return cudaGetLastError();
}
cudaError_t assemble(int N, const double *pw, const double *pn1, const int *perm, double *pi, int grid,
                     cudaStream_t s) {
    PermArg pa;
    for (int u = 0; u < 32; u++) pa.p[u] = u < N ? perm[u] : 0;
    hq2::k_assemble2<<<grid, 256, 0, s>>>(N, pw, pn1, pa, pi);
    return cudaGetLastError();
}

}  // namespace hq2_launch
