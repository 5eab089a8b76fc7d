// hq_batch.cu -- batched solver for many small instances:
// one CTA per instance, the instance's whole state space on chip.  Product code only.
//
// The paper's own usage is many small solves: load sweeps of 9 values per N
// and screening of thousands of location / dispatch configurations of N = 9-11 units
// (PAPER.md:774-931).  hq_batch_solve runs Algorithm 1 literally -- layers
// n = 1..N-1 in order within a sweep, Eq. updateHeter with the inner normalisation limit
// (reading R1), Eqs. lambdaHeter / muHeter after each layer -- for B instances of the same N and J
// at once:
//   * k_batch_dispatch: Wd[b][m][i] = sum_j lambda_j [i is the first free unit of zeta_j in m]
//     (Algorithm 3's dispatch rates, by a scan of the lists) for every state;
//     the upward rate into m through unit i is W_i(m) = Wd[m - i][i] (Eq. tran_rates,
//     PAPER.md:166-175) and lambda_m = sum_i Wd[m][i].  Stays in L2.
//   * k_batch_solve: per CTA, p_n(B_m) (8 B/state), lambda_m, mu_m and the per-layer scratch in
//     shared memory; per layer two block reductions (fixed order: bitwise reproducible); the
//     relative balance residual r(pi) (reading R3) every `check` sweeps; stops at r <= tol.
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <string>
#include <vector>
#include "../../include/hq.h"

namespace hqb {

constexpr int kThreads = 256;
constexpr int kMaxN = 12;

struct BArgs {
    int N, J, B;
    const double *lam;       // [B][J]
    const double *nu;        // [B][N]
    const int32_t *pref;     // [B][J][N], -1 padded
    const double *Wd;        // [B][2^N][N]
    const uint16_t *order;   // [2^N] states sorted by popcount, then value
    int off[kMaxN + 2];      // layer n occupies order[off[n] .. off[n+1])
    double tol;
    int max_iter;
    int check;               // residual every `check` sweeps
    int maxc;                // largest layer, C(N, N/2): size of the x / y scratch
    double *pi;              // [B][2^N] natural index
    int *iters;              // [B]
    double *res;             // [B]
    int *err;                // [B] 0 ok, 1 numeric
    double *workload;        // [B][N] or NULL: rho_i = P(unit i busy)
    double *dispatch;        // [B][J][N] or NULL: rho_ij
    double *loss;            // [B] or NULL
};

__global__ void k_batch_dispatch(BArgs a, double *Wd) {
    const int N = a.N, J = a.J;
    const uint64_t S = 1ull << N, total = S * (uint64_t)a.B;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = t >> N;
        const uint32_t m = (uint32_t)(t & (S - 1));
        double w[kMaxN];
        for (int i = 0; i < N; i++) w[i] = 0.0;
        const double *lam = a.lam + b * J;
        const int32_t *pref = a.pref + b * (uint64_t)J * N;
        for (int j = 0; j < J; j++) {
            const int32_t *row = pref + (uint64_t)j * N;
            for (int h = 0; h < N; h++) {
                const int u = row[h];
                if (u < 0) break;              // list exhausted: the call is lost
                if (!((m >> u) & 1u)) {        // first free unit of the list serves the call
#pragma unroll
                    for (int i = 0; i < kMaxN; i++)
                        if (i == u) w[i] += lam[j];
                    break;
                }
            }
        }
        double *dst = Wd + t * N;
        for (int i = 0; i < N; i++) dst[i] = w[i];
    }
}

// fixed-order block sum of two values (every thread gets the result)
__device__ __forceinline__ double2 block_sum2(double x, double y, double2 *scr) {
    for (int o = 16; o > 0; o >>= 1) {
        x += __shfl_xor_sync(0xffffffffu, x, o);
        y += __shfl_xor_sync(0xffffffffu, y, o);
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();   // scr may still be read from the previous call
    if ((threadIdx.x & 31) == 0) scr[w] = make_double2(x, y);
    __syncthreads();
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < nw; k++) {
        s.x += scr[k].x;
        s.y += scr[k].y;
    }
    return s;
}

__global__ void __launch_bounds__(kThreads) k_batch_solve(BArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int N = a.N, tid = threadIdx.x;
    const uint32_t S = 1u << N;
    double *p = reinterpret_cast<double *>(smem);   // p_n(B_m), natural index
    double *lamm = p + S;                            // lambda_m
    double *mum = lamm + S;                          // mu_m
    double *xs = mum + S;                            // per-layer scratch x_m, y_m (layer-local order)
    double *ys = xs + a.maxc;
    __shared__ double2 scr[kThreads / 32];
    __shared__ double s_lam[kMaxN + 2], s_mu[kMaxN + 2], s_nu[kMaxN], s_pn[kMaxN + 2];

    for (int b = blockIdx.x; b < a.B; b += gridDim.x) {
        const double *Wd = a.Wd + (uint64_t)b * S * N;
        if (tid < N) s_nu[tid] = a.nu[(uint64_t)b * N + tid];
        __syncthreads();
        for (uint32_t m = tid; m < S; m += blockDim.x) {
            double l = 0.0, u = 0.0;
            for (int i = 0; i < N; i++) {
                l += Wd[(uint64_t)m * N + i];
                if ((m >> i) & 1u) u += s_nu[i];
            }
            lamm[m] = l;
            mum[m] = u;
        }
        __syncthreads();
        // Algorithm 1 step 2: uniform conditional probabilities, lambda(n), mu(n) from them
        for (int n = 0; n <= N; n++) {
            const int o0 = a.off[n], o1 = a.off[n + 1];
            const double v = 1.0 / (double)(o1 - o0);
            double sl = 0.0, sm = 0.0;
            for (int k = o0 + tid; k < o1; k += blockDim.x) {
                const uint32_t m = a.order[k];
                p[m] = v;
                sl += v * lamm[m];
                sm += v * mum[m];
            }
            const double2 t = block_sum2(sl, sm, scr);
            if (tid == 0) {
                s_lam[n] = t.x;
                s_mu[n] = t.y;
            }
        }
        __syncthreads();
        int it = 0, bad = 0;
        double r = INFINITY;
        while (true) {
            // one sweep: layers 1..N-1 in order (Algorithm 1 steps 3-9)
            for (int n = 1; n <= N - 1; n++) {
                const int o0 = a.off[n], o1 = a.off[n + 1];
                const double lprev = s_lam[n - 1], beta = s_lam[n] / s_mu[n + 1];
                double sx = 0.0, sy = 0.0;
                for (int k = o0 + tid; k < o1; k += blockDim.x) {
                    const uint32_t m = a.order[k];
                    double A = 0.0, D = 0.0;
                    for (int i = 0; i < N; i++) {
                        const uint32_t bit = 1u << i;
                        if (m & bit) A += p[m ^ bit] * Wd[(uint64_t)(m ^ bit) * N + i];   // from layer n-1
                        else D += p[m | bit] * s_nu[i];                                    // from layer n+1
                    }
                    const double den = lamm[m] + mum[m];
                    const double x = A / (lprev * den), y = beta * D / den;
                    xs[k - o0] = x;
                    ys[k - o0] = y;
                    sx += x;
                    sy += y;
                }
                const double2 t = block_sum2(sx, sy, scr);
                const double mstar = (1.0 - t.y) / t.x;   // the inner loop's limit (reading R1)
                if (!(mstar > 0.0) || !isfinite(mstar)) bad = 1;
                double sl = 0.0, sm = 0.0;
                for (int k = o0 + tid; k < o1; k += blockDim.x) {
                    const uint32_t m = a.order[k];
                    const double v = mstar * xs[k - o0] + ys[k - o0];
                    p[m] = v;
                    sl += v * lamm[m];
                    sm += v * mum[m];
                }
                const double2 u = block_sum2(sl, sm, scr);   // Eqs. lambdaHeter, muHeter
                if (tid == 0) {
                    s_lam[n] = u.x;
                    s_mu[n] = u.y;
                }
                __syncthreads();
            }
            it++;
            const bool last = bad || it >= a.max_iter;
            if (!(last || (a.tol > 0.0 && it % a.check == 0))) continue;
            // p(n) by Eq. bnd_stationary, then the relative balance residual of pi
            if (tid == 0) {
                double prod = 1.0, tot = 1.0;
                s_pn[0] = 1.0;
                for (int n = 1; n <= N; n++) {
                    prod *= s_lam[n - 1] / s_mu[n];
                    s_pn[n] = prod;
                    tot += prod;
                }
                for (int n = 0; n <= N; n++) s_pn[n] /= tot;
            }
            __syncthreads();
            double num = 0.0, dsum = 0.0;
            for (uint32_t m = tid; m < S; m += blockDim.x) {
                double in = 0.0;
                for (int i = 0; i < N; i++) {
                    const uint32_t bit = 1u << i, l = m ^ bit;
                    const double pil = s_pn[__popc(l)] * p[l];
                    if (m & bit) in += pil * Wd[(uint64_t)l * N + i];
                    else in += pil * s_nu[i];
                }
                const double out = s_pn[__popc(m)] * p[m] * (lamm[m] + mum[m]);
                num += fabs(out - in);
                dsum += out;
            }
            const double2 t = block_sum2(num, dsum, scr);
            r = t.x / t.y;
            if (!isfinite(r)) bad = 1;
            if (bad || last || r <= a.tol) break;
        }
        double *out = a.pi + (uint64_t)b * S;
        for (uint32_t m = tid; m < S; m += blockDim.x) out[m] = s_pn[__popc(m)] * p[m];
        if (tid == 0) {
            a.iters[b] = it;
            a.res[b] = r;
            a.err[b] = bad;
        }
        if (a.workload || a.dispatch || a.loss) {
            // measures (as k_measures of the single-instance path): superset sums
            // g(T) = sum_{m superset of T} pi(m) by an in-place zeta transform (fixed order), then
            //   rho_i = g({i}),  loss = sum_j f_j g(list_j),
            //   rho_ij = f_j (g(units before i in zeta_j) - g(units through i)) / (1 - loss)
            double *g = mum;   // mu_m is rebuilt for the next instance
            for (uint32_t m = tid; m < S; m += blockDim.x) g[m] = s_pn[__popc(m)] * p[m];
            for (int bit = 0; bit < N; bit++) {
                __syncthreads();
                for (uint32_t k = tid; k < (S >> 1); k += blockDim.x) {
                    const uint32_t lo = k & ((1u << bit) - 1u), m = ((k >> bit) << (bit + 1)) | lo;
                    g[m] += g[m | (1u << bit)];
                }
            }
            __syncthreads();
            const double *lam = a.lam + (uint64_t)b * a.J;
            const int32_t *pref = a.pref + (uint64_t)b * a.J * N;
            double Lam = 0.0;
            for (int j = 0; j < a.J; j++) Lam += lam[j];
            double lp = 0.0;   // per-thread part of the loss, atoms tid, tid + blockDim, ...
            for (int j = tid; j < a.J; j += blockDim.x) {
                uint32_t T = 0;
                for (int h = 0; h < N && pref[(uint64_t)j * N + h] >= 0; h++) T |= 1u << pref[(uint64_t)j * N + h];
                lp += lam[j] / Lam * g[T];
            }
            const double2 L = block_sum2(lp, 0.0, scr);
            const double loss = L.x;
            if (a.loss && tid == 0) a.loss[b] = loss;
            if (a.workload)
                for (int i = tid; i < N; i += blockDim.x) a.workload[(uint64_t)b * N + i] = g[1u << i];
            if (a.dispatch)
                for (int j = tid; j < a.J; j += blockDim.x) {
                    double *row = a.dispatch + ((uint64_t)b * a.J + j) * N;
                    for (int i = 0; i < N; i++) row[i] = 0.0;
                    const double f = lam[j] / Lam;
                    uint32_t T = 0;
                    for (int h = 0; h < N; h++) {
                        const int u = pref[(uint64_t)j * N + h];
                        if (u < 0) break;
                        const uint32_t T2 = T | (1u << u);
                        row[u] = f * (g[T] - g[T2]) / (1.0 - loss);
                        T = T2;
                    }
                }
        }
        __syncthreads();
    }
}

}  // namespace hqb

void hq_pool_init();   // hq_api.cu: release threshold of the default memory pool

namespace {
thread_local std::string g_batch_error;

hq_status batch_fail(const std::string &m, hq_status st = HQ_E_INVAL) {
    g_batch_error = m;
    return st;
}
}  // namespace

extern "C" const char *hq_batch_error_string(void) { return g_batch_error.c_str(); }

extern "C" hq_status hq_batch_solve(int B, int N, int J, const double *lambda, const double *mu, const int32_t *pref,
                                    double tol, int max_iter, double *pi, void *cuda_stream, int *iters_out,
                                    double *residual_out, int *status_out, double *workload, double *dispatch,
                                    double *loss_out) {
    if (B < 1 || N < 1 || N > hqb::kMaxN || J < 1) return batch_fail("need B >= 1, 1 <= N <= 12, J >= 1");
    if (!lambda || !mu || !pref || !pi) return batch_fail("NULL argument");
    if (max_iter < 1 || !(tol == tol)) return batch_fail("max_iter must be >= 1 and tol not NaN");
    // validation (as hq_create, per instance)
    for (int b = 0; b < B; b++) {
        const double *lam = lambda + (size_t)b * J;
        const double *nu = mu + (size_t)b * N;
        const int32_t *pr = pref + (size_t)b * J * N;
        double L = 0.0;
        for (int j = 0; j < J; j++) {
            if (!std::isfinite(lam[j]) || lam[j] < 0.0) return batch_fail("instance " + std::to_string(b) + ": lambda");
            L += lam[j];
        }
        if (!(L > 0.0)) return batch_fail("instance " + std::to_string(b) + ": sum of lambda must be > 0");
        for (int i = 0; i < N; i++)
            if (!std::isfinite(nu[i]) || !(nu[i] > 0.0)) return batch_fail("instance " + std::to_string(b) + ": mu");
        char reach[hqb::kMaxN] = {0};
        for (int j = 0; j < J; j++) {
            char seen[hqb::kMaxN] = {0};
            bool ended = false;
            int len = 0;
            for (int h = 0; h < N; h++) {
                const int u = pr[(size_t)j * N + h];
                if (u == -1) {
                    ended = true;
                    continue;
                }
                if (ended || u < 0 || u >= N || seen[u])
                    return batch_fail("instance " + std::to_string(b) + ": invalid preference row " + std::to_string(j));
                seen[u] = 1;
                len++;
                if (lam[j] > 0.0) reach[u] = 1;
            }
            if (len == 0) return batch_fail("instance " + std::to_string(b) + ": empty preference row");
        }
        for (int i = 0; i < N; i++)
            if (!reach[i]) return batch_fail("instance " + std::to_string(b) + ": reducible chain (unit in no list)");
    }
    cudaStream_t s = (cudaStream_t)cuda_stream;
    hq_pool_init();
    const uint32_t S = 1u << N;
    hqb::BArgs a;
    memset(&a, 0, sizeof(a));
    a.N = N;
    a.J = J;
    a.B = B;
    a.tol = tol;
    a.max_iter = max_iter;
    a.check = 4;
    std::vector<uint16_t> order;
    order.reserve(S);
    for (int n = 0; n <= N; n++) {
        a.off[n] = (int)order.size();
        for (uint32_t m = 0; m < S; m++)
            if (__builtin_popcount(m) == n) order.push_back((uint16_t)m);
    }
    a.off[N + 1] = (int)S;
    double *d_lam = nullptr, *d_nu = nullptr, *d_Wd = nullptr, *d_res = nullptr;
    int32_t *d_pref = nullptr;
    uint16_t *d_order = nullptr;
    int *d_it = nullptr, *d_err = nullptr;
    double *d_loss = nullptr;
    auto cleanup = [&]() {   // stream-ordered frees (the default pool recycles the blocks)
        if (d_lam) cudaFreeAsync(d_lam, s);
        if (d_nu) cudaFreeAsync(d_nu, s);
        if (d_Wd) cudaFreeAsync(d_Wd, s);
        if (d_res) cudaFreeAsync(d_res, s);
        if (d_pref) cudaFreeAsync(d_pref, s);
        if (d_order) cudaFreeAsync(d_order, s);
        if (d_it) cudaFreeAsync(d_it, s);
        if (d_err) cudaFreeAsync(d_err, s);
        if (d_loss) cudaFreeAsync(d_loss, s);
    };
#define HQB_CUDA(x)                                                                          \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess) {                                                             \
            cleanup();                                                                       \
            return batch_fail(std::string("CUDA error: ") + cudaGetErrorString(e_), HQ_E_CUDA); \
        }                                                                                    \
    } while (0)
    HQB_CUDA(cudaMallocAsync((void **)&d_lam, sizeof(double) * B * J, s));
    HQB_CUDA(cudaMallocAsync((void **)&d_nu, sizeof(double) * B * N, s));
    HQB_CUDA(cudaMallocAsync((void **)&d_pref, sizeof(int32_t) * B * J * N, s));
    HQB_CUDA(cudaMallocAsync((void **)&d_Wd, sizeof(double) * (size_t)B * S * N, s));
    HQB_CUDA(cudaMallocAsync((void **)&d_order, sizeof(uint16_t) * S, s));
    HQB_CUDA(cudaMallocAsync((void **)&d_res, sizeof(double) * B, s));
    HQB_CUDA(cudaMallocAsync((void **)&d_it, sizeof(int) * B, s));
    HQB_CUDA(cudaMallocAsync((void **)&d_err, sizeof(int) * B, s));
    HQB_CUDA(cudaMemcpyAsync(d_lam, lambda, sizeof(double) * B * J, cudaMemcpyHostToDevice, s));
    HQB_CUDA(cudaMemcpyAsync(d_nu, mu, sizeof(double) * B * N, cudaMemcpyHostToDevice, s));
    HQB_CUDA(cudaMemcpyAsync(d_pref, pref, sizeof(int32_t) * B * J * N, cudaMemcpyHostToDevice, s));
    HQB_CUDA(cudaMemcpyAsync(d_order, order.data(), sizeof(uint16_t) * S, cudaMemcpyHostToDevice, s));
    a.lam = d_lam;
    a.nu = d_nu;
    a.pref = d_pref;
    a.Wd = d_Wd;
    a.order = d_order;
    a.pi = pi;
    a.iters = d_it;
    a.res = d_res;
    a.err = d_err;
    a.workload = workload;
    a.dispatch = dispatch;
    if (loss_out) {
        HQB_CUDA(cudaMallocAsync((void **)&d_loss, sizeof(double) * B, s));
        a.loss = d_loss;
    }
    int dev = 0, nsm = 148;
    HQB_CUDA(cudaGetDevice(&dev));
    HQB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    hqb::k_batch_dispatch<<<nsm * 8, 256, 0, s>>>(a, d_Wd);
    HQB_CUDA(cudaGetLastError());
    for (int n = 0; n <= N; n++) a.maxc = std::max(a.maxc, a.off[n + 1] - a.off[n]);
    const size_t sm = sizeof(double) * (3 * (size_t)S + 2 * (size_t)a.maxc);
    HQB_CUDA(cudaFuncSetAttribute(hqb::k_batch_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int per_sm = 1;
    const int nthr = S <= 256 ? 64 : S <= 1024 ? 128 : hqb::kThreads;   // small state spaces: more, smaller CTAs (measured)
    HQB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hqb::k_batch_solve, nthr, sm));
    const int grid = std::min(B, nsm * std::max(1, per_sm));
    hqb::k_batch_solve<<<grid, nthr, sm, s>>>(a);
    HQB_CUDA(cudaGetLastError());
    std::vector<int> it(B), er(B);
    std::vector<double> rr(B);
    HQB_CUDA(cudaMemcpyAsync(it.data(), d_it, sizeof(int) * B, cudaMemcpyDeviceToHost, s));
    HQB_CUDA(cudaMemcpyAsync(rr.data(), d_res, sizeof(double) * B, cudaMemcpyDeviceToHost, s));
    HQB_CUDA(cudaMemcpyAsync(er.data(), d_err, sizeof(int) * B, cudaMemcpyDeviceToHost, s));
    if (loss_out) HQB_CUDA(cudaMemcpyAsync(loss_out, d_loss, sizeof(double) * B, cudaMemcpyDeviceToHost, s));
    HQB_CUDA(cudaStreamSynchronize(s));
    cleanup();
    hq_status worst = HQ_OK;
    for (int b = 0; b < B; b++) {
        hq_status sb = er[b] ? HQ_E_NUMERIC : (tol > 0.0 && !(rr[b] <= tol)) ? HQ_NOT_CONVERGED : HQ_OK;
        if (status_out) status_out[b] = sb;
        if (iters_out) iters_out[b] = it[b];
        if (residual_out) residual_out[b] = rr[b];
        if (sb == HQ_E_NUMERIC) worst = HQ_E_NUMERIC;
        else if (sb == HQ_NOT_CONVERGED && worst == HQ_OK) worst = HQ_NOT_CONVERGED;
    }
    if (worst == HQ_E_NUMERIC) g_batch_error = "non-positive or non-finite layer normaliser in some instance";
    return worst;
#undef HQB_CUDA
}
