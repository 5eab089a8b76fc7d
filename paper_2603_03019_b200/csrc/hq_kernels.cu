// hq_kernels.cu -- sm_100a kernels of the B200 hypercube-queue solver.
//
// Every kernel walks the parity-compressed state space (hq_internal.h) in
// tiles of HQ_BLOCK * R consecutive compressed indices; a persistent grid
// strides over the tiles.  Per-layer sums are reduced deterministically:
// per-thread register bins keyed by popcount(r), a fixed-order shared-memory
// transpose-reduce keyed by popcount(j), one partial row per CTA, and a
// fixed-order final reduction (k_layer_reduce).  No floating-point atomics.
//
// Paper passages:
//   gather      Eq. updateHeter (313-315): p_n(m) = mu(n)/lambda(n-1) A(m)/den(m)
//               + lambda(n)/mu(n+1) D(m)/den(m), den = lambda_m + mu_m;
//               upward rates lambda_lm of Eq. tran_rates (166-175) are computed
//               on the fly from the preference trie (Algorithm 3 semantics,
//               541-567, read with SURVEY.md C6).
//   reduce      Eqs. lambdaHeter / muHeter (318-319) and the inner fixed point
//               of Algorithm 1 (343-348) in closed form mu* = (1 - sum b)/sum a
//               (reading R1).
//   residual    Eq. balance_eq_heter (161) as a relative L1 residual (R3).
//   assemble    Proposition 1 (224) + Eq. bnd_stationary (227).
//   measures    rho_i and rho_ij (787-789, 1757-1761) via superset sums.
#include <cuda_runtime.h>
#include <cstdint>
#include "hq_internal.h"

namespace hqk {

template <int R> struct Log2 { static constexpr int v = 1 + Log2<R / 2>::v; };
template <> struct Log2<1> { static constexpr int v = 0; };

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// ---------------------------------------------------------------------------
// On-the-fly rates (v1: per-thread preorder walk of the preference trie).
//   A    = sum over busy u of W_u(m) * q[m ^ e_u],  W_u(m) = lambda_{m\u -> m}
//   D    = sum over free u of nu_u * q[m ^ e_u]
//   lam  = lambda_m (Lambda minus the atoms whose whole list is busy)
//   mu   = mu_m = sum of nu_u over busy u
// q is the neighbour class array at compressed indices.
// ---------------------------------------------------------------------------
struct Gathered {
    double A, D, lam, mu;
};

__device__ __forceinline__ Gathered gather_state(const KArgs &k, uint32_t j, uint32_t m, const double *__restrict__ q) {
    double W[HQ_MAXN + 1];
#pragma unroll
    for (int u = 0; u < HQ_MAXN + 1; u++) W[u] = 0.0;
    double blocked = 0.0;
    const int2 *__restrict__ node = k.trie.node;
    const double *__restrict__ lthr = k.trie.lam_thr;
    const double *__restrict__ lend = k.trie.lam_end;
    int v = 0;
    const int nn = k.trie.nnodes;
    while (v < nn) {
        int2 nd = __ldg(&node[v]);
        const int nu_ = nd.x & 0xff;
        if ((m >> nu_) & 1u) {
            W[nu_] += __ldg(&lthr[v]);
            if (!k.full_lists) blocked += __ldg(&lend[v]);
            v++;
        } else {
            v = nd.y;
        }
    }
    Gathered g;
    g.A = 0.0;
    g.D = 0.0;
    g.mu = 0.0;
    for (int u = 0; u < k.N; u++) {
        uint32_t jn = u ? (j ^ (1u << (u - 1))) : j;
        double qv = __ldg(&q[jn]);
        if ((m >> u) & 1u) {
            g.A = fma(W[u], qv, g.A);
            g.mu += k.nu[u];
        } else {
            g.D = fma(k.nu[u], qv, g.D);
        }
    }
    g.lam = k.full_lists ? (m == (1u << k.N) - 1u ? 0.0 : k.Lam) : (k.Lam - blocked);
    return g;
}

// ---------------------------------------------------------------------------
// Generic persistent tile loop with deterministic per-layer reduction.
// per_state(j, vals) returns true if the state contributes vals[0..NV).
// Results: partial[blockIdx][n][v] for layer n (layers are derived from the
// popcount of j and the class c).
// ---------------------------------------------------------------------------
template <int R, int NV, class F>
__device__ __forceinline__ void tile_loop(const KArgs &k, double *__restrict__ partial, F per_state) {
    constexpr int KB = Log2<R>::v + 1;
    extern __shared__ double red[];            // [KB][NV][HQ_BLOCK]
    __shared__ double sacc[HQ_NL][NV];         // keyed by popcount(j)
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < HQ_NL * NV; i += HQ_BLOCK) (&sacc[0][0])[i] = 0.0;
    __syncthreads();
    const uint64_t tile_states = (uint64_t)HQ_BLOCK * R;
    for (uint64_t tile = blockIdx.x; tile < k.ntiles; tile += gridDim.x) {
        double acc[KB][NV];
#pragma unroll
        for (int b = 0; b < KB; b++)
#pragma unroll
            for (int v = 0; v < NV; v++) acc[b][v] = 0.0;
#pragma unroll
        for (int r = 0; r < R; r++) {
            const uint64_t j = tile * tile_states + (uint64_t)r * HQ_BLOCK + tid;
            if (j < k.nstates_c) {
                double vals[NV];
                if (per_state((uint32_t)j, vals)) {
                    constexpr int dummy = 0;
                    (void)dummy;
                    const int b = __popc(r);
#pragma unroll
                    for (int v = 0; v < NV; v++) acc[b][v] += vals[v];
                }
            }
        }
#pragma unroll
        for (int b = 0; b < KB; b++)
#pragma unroll
            for (int v = 0; v < NV; v++) red[(b * NV + v) * HQ_BLOCK + tid] = acc[b][v];
        __syncthreads();
        const int pcg = __popcll(tile);
        constexpr int NRB = 8 + KB;            // relative bins popcount(tid) + b in [0, 8 + KB - 1]
        for (int o = warp; o < NRB * NV; o += HQ_BLOCK / 32) {
            const int rb = o / NV, v = o % NV;
            double s = 0.0;
            for (int t = lane; t < HQ_BLOCK; t += 32) {
                const int kk = rb - __popc(t);
                if (kk >= 0 && kk < KB) s += red[(kk * NV + v) * HQ_BLOCK + t];
            }
            s = warp_sum(s);
            if (lane == 0 && pcg + rb < HQ_NL) sacc[pcg + rb][v] += s;
        }
        __syncthreads();
    }
    // popcount(j) -> layer n = pc + (c ^ (pc & 1)); layer n collects pc = n-1 and pc = n
    double *out = partial + (size_t)blockIdx.x * HQ_NL * HQ_NV;
    for (int i = tid; i < HQ_NL * NV; i += HQ_BLOCK) {
        const int n = i / NV, v = i % NV;
        double s = 0.0;
        if ((n & 1) == k.c) {
            if (n >= 1) s += sacc[n - 1][v];
            s += sacc[n][v];
        }
        out[n * HQ_NV + v] = s;
    }
}

__device__ __forceinline__ void decode(const KArgs &k, uint32_t j, int &n, uint32_t &m) {
    const int pc = __popc(j);
    const int b0 = k.c ^ (pc & 1);
    n = pc + b0;
    m = (j << 1) | (uint32_t)b0;
}

// ---------------------------------------------------------------------------
// Gather: a_m, b_m of Eq. updateHeter for every state of the active layers.
// ---------------------------------------------------------------------------
template <int R>
__global__ void __launch_bounds__(HQ_BLOCK) k_gather(KArgs k) {
    tile_loop<R, 6>(k, k.partial, [&](uint32_t j, double *vals) -> bool {
        int n;
        uint32_t m;
        decode(k, j, n, m);
        if (!((k.active >> n) & 1u)) return false;
        Gathered g = gather_state(k, j, m, k.Q);
        const double den = g.lam + g.mu;
        const double a = g.A / (k.lam_n[n - 1] * den);
        const double b = (k.lam_n[n] / k.mu_n[n + 1]) * g.D / den;
        k.ab[j] = make_double2(a, b);
        vals[RV_SA] = a;
        vals[RV_SB] = b;
        vals[RV_SLA] = g.lam * a;
        vals[RV_SLB] = g.lam * b;
        vals[RV_SMA] = g.mu * a;
        vals[RV_SMB] = g.mu * b;
        return true;
    });
}

// Finalize: p_n(m) = mu*(n) a_m + b_m (in place), per-layer |dp| and sum p.
template <int R>
__global__ void __launch_bounds__(HQ_BLOCK) k_finalize(KArgs k) {
    tile_loop<R, 3>(k, k.partial, [&](uint32_t j, double *vals) -> bool {
        int n;
        uint32_t m;
        decode(k, j, n, m);
        if (!((k.active >> n) & 1u)) return false;
        const double2 ab = k.ab[j];
        const double pnew = fma(k.mustar[n], ab.x, ab.y);
        const double pold = k.P[j];
        k.P[j] = pnew;
        vals[FV_DL1] = fabs(pnew - pold);
        vals[FV_DDEN] = 0.0;
        vals[FV_SUMP] = pnew;
        return true;
    });
}

// Init: p_n(m) = 1/C(N,n) for every state of class c (Algorithm 1 step 2,
// PAPER.md:337) and the layer sums of lambda_m p and mu_m p (Eqs.
// lambdaHeter / muHeter on the uniform p, reading R8).  k.mustar holds
// 1/C(N,n) here.
template <int R>
__global__ void __launch_bounds__(HQ_BLOCK) k_init(KArgs k) {
    tile_loop<R, 2>(k, k.partial, [&](uint32_t j, double *vals) -> bool {
        int n;
        uint32_t m;
        decode(k, j, n, m);
        const double p = k.mustar[n];
        k.P[j] = p;
        double lam, mu = 0.0;
        if (k.full_lists) {
            lam = (n == k.N) ? 0.0 : k.Lam;
        } else {
            // lambda_m: atoms with every listed unit busy are lost (trie walk)
            double blocked = 0.0;
            int v = 0;
            while (v < k.trie.nnodes) {
                int2 nd = k.trie.node[v];
                if ((m >> (nd.x & 0xff)) & 1u) {
                    blocked += k.trie.lam_end[v];
                    v++;
                } else {
                    v = nd.y;
                }
            }
            lam = k.Lam - blocked;
        }
        for (int u = 0; u < k.N; u++)
            if ((m >> u) & 1u) mu += k.nu[u];
        vals[0] = lam * p;
        vals[1] = mu * p;
        return true;
    });
}

// v2 init: p_n(m) = 1/C(N,n) and the layer sums {p, p mu_m, p omega, p kappa,
// p lambda_m} that seed the a-priori normalisation of the first half-sweep.
template <int R>
__global__ void __launch_bounds__(HQ_BLOCK) k_init_v2(KArgs k) {
    tile_loop<R, 5>(k, k.partial, [&](uint32_t j, double *vals) -> bool {
        int n;
        uint32_t m;
        decode(k, j, n, m);
        const double p = k.mustar[n];
        k.P[j] = p;
        double lam;
        if (k.full_lists) lam = (n == k.N) ? 0.0 : k.Lam;
        else lam = k.lamarr[j];
        double mu = 0.0;
        for (int u = 0; u < k.N; u++)
            if ((m >> u) & 1u) mu += k.nu[u];
        const double2 ok = k.omkap[j];
        vals[0] = p;
        vals[1] = p * mu;
        vals[2] = p * ok.x;
        vals[3] = p * ok.y;
        vals[4] = p * lam;
        return true;
    });
}

// Residual (reading R3) for the states of class c: |outflow - inflow| and
// outflow of Eq. balance_eq_heter with pi(m) = p(n) p_n(m).
template <int R>
__global__ void __launch_bounds__(HQ_BLOCK) k_residual(KArgs k) {
    tile_loop<R, 2>(k, k.partial, [&](uint32_t j, double *vals) -> bool {
        int n;
        uint32_t m;
        decode(k, j, n, m);
        Gathered g = gather_state(k, j, m, k.Q);
        const double pm = k.pn[n] * k.P[j];
        const double out = pm * (g.lam + g.mu);
        const double lo = n >= 1 ? k.pn[n - 1] : 0.0;
        const double hi = n + 1 <= k.N ? k.pn[n + 1] : 0.0;
        const double in = lo * g.A + hi * g.D;
        vals[0] = fabs(out - in);
        vals[1] = out;
        return true;
    });
}

// ---------------------------------------------------------------------------
// Layer reduction: one warp per layer sums the CTA partials in fixed order.
//   mode 0 (after gather): mu*(n) = (1 - sum b)/sum a; lambda(n), mu(n).
//   mode 1 (after finalize): per-layer |dp| and sum p into stats.
//   mode 2 (after init, both classes): lambda(n), mu(n).
//   mode 3 (after residual, both classes): totals into stats.
// ---------------------------------------------------------------------------
struct ReduceArgs {
    int N;
    uint32_t active;
    int ncta;
    int nbuf;                // number of partial buffers (classes) to add
    const double *partial;   // [nbuf][ncta][HQ_NL][HQ_NV]
    int NV;
    int mode;
    double *lam_n, *mu_n, *mustar;
    double *stats;           // [HQ_NL][4]
    int *err;
};

__global__ void __launch_bounds__(1024) k_layer_reduce(ReduceArgs a) {
    const int lane = threadIdx.x & 31, n = threadIdx.x >> 5;
    if (n > a.N) return;
    double s[HQ_NV];
    for (int v = 0; v < a.NV; v++) s[v] = 0.0;
    for (int b = 0; b < a.nbuf; b++) {
        const double *P = a.partial + (size_t)b * a.ncta * HQ_NL * HQ_NV;
        for (int i = lane; i < a.ncta; i += 32)
            for (int v = 0; v < a.NV; v++) s[v] += P[((size_t)i * HQ_NL + n) * HQ_NV + v];
    }
    for (int v = 0; v < a.NV; v++) s[v] = warp_sum(s[v]);
    if (lane != 0) return;
    if (a.mode == 0) {
        if (!((a.active >> n) & 1u)) return;
        const double sa = s[RV_SA], sb = s[RV_SB];
        const double ms = (1.0 - sb) / sa;
        if (!(sa > 0.0) || !isfinite(ms)) atomicExch(a.err, 1);
        a.mustar[n] = ms;
        a.lam_n[n] = fma(ms, s[RV_SLA], s[RV_SLB]);
        a.mu_n[n] = fma(ms, s[RV_SMA], s[RV_SMB]);
    } else if (a.mode == 1) {
        if (!((a.active >> n) & 1u)) return;
        a.stats[n * 4 + 0] = s[FV_DL1];
        a.stats[n * 4 + 1] = s[FV_SUMP];
    } else if (a.mode == 2) {
        a.lam_n[n] = s[0];
        a.mu_n[n] = s[1];
    } else {
        a.stats[n * 4 + 2] = s[0];
        a.stats[n * 4 + 3] = s[1];
    }
}

// pi[m] = p(w(m)) * p_{w(m)}(m) at natural index m (Proposition 1).
__global__ void k_assemble(int N, const double *__restrict__ pw, const double *__restrict__ pn, double *__restrict__ pi) {
    const uint64_t S = 1ull << N, half = S >> 1;
    for (uint64_t m = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; m < S; m += (uint64_t)gridDim.x * blockDim.x) {
        const int n = __popcll(m);
        const uint64_t off = (n & 1) ? half : 0;
        pi[m] = pn[n] * pw[off + (m >> 1)];
    }
}

// Superset sums g(S) = sum_{m >= S} pi(m), one bit per launch.
__global__ void k_zeta_bit(int N, int bit, double *__restrict__ g) {
    const uint64_t half = 1ull << (N - 1);
    const uint64_t lowmask = (1ull << bit) - 1;
    for (uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s < half; s += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t idx = ((s & ~lowmask) << 1) | (s & lowmask);
        g[idx] += g[idx | (1ull << bit)];
    }
}

// Measures from superset sums (one thread block; J*N is small).
//   loss    = sum_j f_j g(list_j)
//   rho_i   = g({i})
//   rho_ij  = f_j (g(prefix before i) - g(prefix through i)) / (1 - loss)
__global__ void k_measures(int N, int J, const double *__restrict__ lam, double Lam, const int32_t *__restrict__ pref,
                           const double *__restrict__ g, double *__restrict__ workload, double *__restrict__ dispatch,
                           double *__restrict__ loss_out) {
    __shared__ double sl[1024];
    __shared__ double s_loss;
    double part = 0.0;
    for (int j = threadIdx.x; j < J; j += blockDim.x) {
        uint64_t mask = 0;
        for (int h = 0; h < N; h++) {
            const int u = pref[(size_t)j * N + h];
            if (u < 0) break;
            mask |= 1ull << u;
        }
        part += (lam[j] / Lam) * g[mask];
    }
    sl[threadIdx.x] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < (int)blockDim.x; i++) s += sl[i];
        s_loss = s;
        *loss_out = s;
    }
    __syncthreads();
    const double loss = s_loss;
    for (int i = threadIdx.x; i < N; i += blockDim.x) workload[i] = g[1ull << i];
    for (int j = threadIdx.x; j < J; j += blockDim.x) {
        const double fj = lam[j] / Lam;
        for (int i = 0; i < N; i++) dispatch[(size_t)j * N + i] = 0.0;
        uint64_t mask = 0;
        for (int h = 0; h < N; h++) {
            const int u = pref[(size_t)j * N + h];
            if (u < 0) break;
            const double before = g[mask];
            mask |= 1ull << u;
            dispatch[(size_t)j * N + u] = fj * (before - g[mask]) / (1.0 - loss);
        }
    }
}

// ---- waiting room (finite buffer C > 0 or unlimited), full preference lists
// (Proposition "Reformulation, Finite Buffer"; Remark).
// The conditional probabilities p_n(B_m) are those of the loss system; the layer masses
// follow the extended birth-death chain, so pi of the hypercube states is the loss-system
// pi scaled by s = 1 / (1 + sum_c G(N + c) / G(N) p(N)).
__global__ void k_scale(double *__restrict__ x, uint64_t n, double s) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        x[i] *= s;
}

// Measures of the queued system from those of the hypercube states (k_measures output):
//   rho_i  += sum_c P~{c}                  (every unit is busy while calls wait)
//   rho_ij  = [f_j sum_{S_ij} pi + f_j P_wait nu_i / sum nu] / (1 - loss_q)
// where P_wait = P(all busy, room in the buffer) and a queued call is served by the unit
// that completes service first (unit i with probability nu_i / sum nu; R14).
__global__ void k_buffer_measures(int N, int J, const double *__restrict__ lam, double Lam, NuArg nu,
                                  const double *__restrict__ pi_all_busy, const double *__restrict__ loss_dev,
                                  double tail_mass, double tail_last, double loss_q, double *__restrict__ workload,
                                  double *__restrict__ dispatch) {
    const double pall = *pi_all_busy, ld = *loss_dev;
    const double pwait = pall + tail_mass - tail_last;
    double snu = 0.0;
    for (int i = 0; i < N; i++) snu += nu.v[i];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < J * N; k += gridDim.x * blockDim.x) {
        const int j = k / N, i = k - j * N;
        const double f = lam[j] / Lam;
        dispatch[k] = (dispatch[k] * (1.0 - ld) + f * pwait * nu.v[i] / snu) / (1.0 - loss_q);
    }
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < N; i += blockDim.x) workload[i] += tail_mass;
}

// Response-time measures from the dispatch
// fractions rho_ij of k_measures: one CTA, atoms over threads, fixed-order sums.
//   MRT_j = sum_i rho_ij tau_ij / sum_i rho_ij,  F_j(T) = sum_{i: tau_ij < T} rho_ij / f_j
//   MRT   = sum_ij rho_ij tau_ij,                F(T)   = sum_{ij: tau_ij < T} rho_ij
// (E(j, T) is the disjoint union of the S_ij with tau_ij < T, so its mass is sum rho_ij (1 - Pi) / f_j.)
__global__ void k_response(int N, int J, const double *__restrict__ lam, double Lam, const double *__restrict__ disp,
                           const double *__restrict__ tau, double T, double *__restrict__ mrt_j,
                           double *__restrict__ f_j, double *__restrict__ tot) {
    __shared__ double s_m[1024], s_f[1024];
    double pm = 0.0, pf = 0.0;
    for (int j = threadIdx.x; j < J; j += blockDim.x) {
        double num = 0.0, den = 0.0, fin = 0.0;
        for (int i = 0; i < N; i++) {
            const double r = disp[(size_t)j * N + i], t = tau[(size_t)j * N + i];
            num += r * t;
            den += r;
            if (t < T) fin += r;
        }
        const double f = lam[j] / Lam;
        if (mrt_j) mrt_j[j] = den > 0.0 ? num / den : 0.0;
        if (f_j) f_j[j] = f > 0.0 ? fin / f : 0.0;
        pm += num;
        pf += fin;
    }
    s_m[threadIdx.x] = pm;
    s_f[threadIdx.x] = pf;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < (int)blockDim.x; k++) {
            a += s_m[k];
            b += s_f[k];
        }
        tot[0] = a;
        tot[1] = b;
    }
}

}  // namespace hqk

// ---------------------------------------------------------------------------
// Launchers (host side, same translation unit).
// ---------------------------------------------------------------------------
namespace hqk_launch {

constexpr int R = 4;

static size_t red_smem(int NV) { return sizeof(double) * (hqk::Log2<R>::v + 1) * NV * HQ_BLOCK; }

cudaError_t gather(const KArgs &k, int grid, cudaStream_t s) {
    hqk::k_gather<R><<<grid, HQ_BLOCK, red_smem(6), s>>>(k);
    return cudaGetLastError();
}
cudaError_t finalize(const KArgs &k, int grid, cudaStream_t s) {
    hqk::k_finalize<R><<<grid, HQ_BLOCK, red_smem(3), s>>>(k);
    return cudaGetLastError();
}
cudaError_t init(const KArgs &k, int grid, cudaStream_t s) {
    hqk::k_init<R><<<grid, HQ_BLOCK, red_smem(2), s>>>(k);
    return cudaGetLastError();
}
cudaError_t init_v2(const KArgs &k, int grid, cudaStream_t s) {
    hqk::k_init_v2<R><<<grid, HQ_BLOCK, red_smem(5), s>>>(k);
    return cudaGetLastError();
}
cudaError_t residual(const KArgs &k, int grid, cudaStream_t s) {
    hqk::k_residual<R><<<grid, HQ_BLOCK, red_smem(2), s>>>(k);
    return cudaGetLastError();
}
cudaError_t layer_reduce(int N, uint32_t active, int ncta, int nbuf, const double *partial, int NV, int mode,
                         double *lam_n, double *mu_n, double *mustar, double *stats, int *err, cudaStream_t s) {
    hqk::ReduceArgs a{N, active, ncta, nbuf, partial, NV, mode, lam_n, mu_n, mustar, stats, err};
    hqk::k_layer_reduce<<<1, 1024, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t assemble(int N, const double *pw, const double *pn, double *pi, int grid, cudaStream_t s) {
    hqk::k_assemble<<<grid, 256, 0, s>>>(N, pw, pn, pi);
    return cudaGetLastError();
}
cudaError_t zeta(int N, double *g, int grid, cudaStream_t s) {
    for (int b = 0; b < N; b++) {
        hqk::k_zeta_bit<<<grid, 256, 0, s>>>(N, b, g);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}
cudaError_t response(int N, int J, const double *lam, double Lam, const double *disp, const double *tau, double T,
                     double *mrt_j, double *f_j, double *tot, cudaStream_t s) {
    hqk::k_response<<<1, 1024, 0, s>>>(N, J, lam, Lam, disp, tau, T, mrt_j, f_j, tot);
    return cudaGetLastError();
}
cudaError_t scale(double *x, uint64_t n, double f, int grid, cudaStream_t s) {
    hqk::k_scale<<<grid, 256, 0, s>>>(x, n, f);
    return cudaGetLastError();
}
cudaError_t buffer_measures(int N, int J, const double *lam, double Lam, const double *nu, const double *pi_all_busy,
                            const double *loss_dev, double tail_mass, double tail_last, double loss_q,
                            double *workload, double *dispatch, cudaStream_t s) {
    NuArg a;
    for (int i = 0; i < 32; i++) a.v[i] = i < N ? nu[i] : 0.0;
    hqk::k_buffer_measures<<<8, 256, 0, s>>>(N, J, lam, Lam, a, pi_all_busy, loss_dev, tail_mass, tail_last, loss_q,
                                             workload, dispatch);
    return cudaGetLastError();
}
cudaError_t measures(int N, int J, const double *lam, double Lam, const int32_t *pref, const double *g,
                     double *workload, double *dispatch, double *loss, cudaStream_t s) {
    hqk::k_measures<<<1, 1024, 0, s>>>(N, J, lam, Lam, pref, g, workload, dispatch, loss);
    return cudaGetLastError();
}
int tile_states() { return HQ_BLOCK * R; }

}  // namespace hqk_launch
