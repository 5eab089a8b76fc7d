// layout_ab.cu -- measurement behind the layout decision of DESIGN.md §4 (north star: "the
// choice between colex-ranked contiguous layers and natural bit indexing is decided by
// measurement").  Development tool, not product code.
//
// Both kernels compute the same layer-gather skeleton of Eq. updateHeter (PAPER.md:313-315,
// the N single-bit-flip neighbours of every state) without the rate programs:
//     out(m) = sum_i c_i(m) x(m xor e_i),   c_i(m) = w_i if i in m else v_i
// over all 2^N states, fp64, one pass; inputs larger than L2 at N >= 24.
//   natural: x and out indexed by the bit pattern m (one thread per state; neighbours
//            m xor 2^i: low bits inside a warp's 256-byte segment, high bits as coalesced
//            streams of another segment)
//   colex:   each layer n stored contiguously in colexicographic rank order
//            (rank(m) = sum_k C(b_k, k) over the set bits b_1 < .. < b_n); a thread owns
//            consecutive ranks of one layer, steps the bit set with Gosper's next-combination,
//            and computes every neighbour's rank from prefix / suffix sums of binomials
//            (removing b_j: S_<j + sum_{k>j} C(b_k, k-1); adding i with j set bits below:
//            S_<=j + C(i, j+1) + sum_{k>j} C(b_k, k+1)).
// The two results are compared state by state (same fp64 summation order over i).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o layout_ab layout_ab.cu
//   ./layout_ab N [reps]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <algorithm>

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));         \
            exit(1);                                                                           \
        }                                                                                      \
    } while (0)

__constant__ double c_w[32], c_v[32];
__constant__ uint64_t c_off[34];      // start of layer n in the colex array
__constant__ uint32_t c_binom[33][34];  // C(x, k), x <= 32, k <= 33

__global__ void k_natural(int N, const double *__restrict__ x, double *__restrict__ out) {
    const uint64_t S = 1ull << N;
    for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < S; m += (uint64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < N; i++) {
            const double c = ((m >> i) & 1) ? c_w[i] : c_v[i];
            s = fma(c, __ldg(x + (m ^ (1ull << i))), s);
        }
        out[m] = s;
    }
}

// colex rank of a bit set
__device__ __forceinline__ uint64_t crank(uint32_t m) {
    uint64_t r = 0;
    int k = 1;
    while (m) {
        const int b = __ffs(m) - 1;
        r += c_binom[b][k++];
        m &= m - 1;
    }
    return r;
}
// colex unrank: the bit set of rank r in layer n
__device__ __forceinline__ uint32_t cunrank(int N, int n, uint64_t r) {
    uint32_t m = 0;
    for (int k = n; k >= 1; k--) {
        int b = k - 1;
        while (b + 1 < N && c_binom[b + 1][k] <= r) b++;
        m |= 1u << b;
        r -= c_binom[b][k];
    }
    return m;
}

// one thread: PER consecutive ranks of layer n
template <int PER>
__global__ void k_colex(int N, const double *__restrict__ x, double *__restrict__ out, const uint64_t *tstart,
                        int nthreads_total) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nthreads_total) return;
    // locate the layer of this thread (tstart[n] = first thread of layer n)
    int n = 0;
    while (n < N && (uint64_t)g >= tstart[n + 1]) n++;
    const uint64_t r0 = ((uint64_t)g - tstart[n]) * PER;
    const uint64_t L = c_binom[N][n];
    if (r0 >= L) return;
    uint32_t m = cunrank(N, n, r0);
    for (int e = 0; e < PER && r0 + e < L; e++) {
        // prefix sums over the set bits b_1 < .. < b_n: P0[j] = sum_{k<=j} C(b_k, k),
        // Pm[j] = sum_{k>j} C(b_k, k-1), Pp[j] = sum_{k>j} C(b_k, k+1)
        int bits[32];
        int nb = 0;
        for (uint32_t t = m; t; t &= t - 1) bits[nb++] = __ffs(t) - 1;
        uint64_t P0[33], Pm[33], Pp[33];
        P0[0] = 0;
        for (int j = 1; j <= nb; j++) P0[j] = P0[j - 1] + c_binom[bits[j - 1]][j];
        Pm[nb] = Pp[nb] = 0;
        for (int j = nb - 1; j >= 0; j--) {
            Pm[j] = Pm[j + 1] + c_binom[bits[j]][j];          // bit k = j + 1 -> C(b, k - 1)
            Pp[j] = Pp[j + 1] + c_binom[bits[j]][j + 2];      // C(b, k + 1)
        }
        double s = 0.0;
        int below = 0;   // set bits below i
        for (int i = 0; i < N; i++) {
            double v;
            if ((m >> i) & 1) {
                // remove bit i = b_{below+1}: layer n-1
                const uint64_t rr = P0[below] + Pm[below + 1];
                v = c_w[i] * __ldg(x + c_off[n - 1] + rr);
                below++;
            } else {
                // add bit i with `below` set bits under it: layer n+1
                const uint64_t rr = P0[below] + c_binom[i][below + 1] + Pp[below];
                v = c_v[i] * __ldg(x + c_off[n + 1] + rr);
            }
            s += v;
        }
        out[c_off[n] + r0 + e] = s;
        // next combination (Gosper)
        const uint32_t c = m & (0u - m), rr = m + c;
        m = (((rr ^ m) >> 2) / c) | rr;
    }
}

// the natural kernel with the same summation as the colex one (product then add)
__global__ void k_natural2(int N, const double *__restrict__ x, double *__restrict__ out) {
    const uint64_t S = 1ull << N;
    for (uint64_t m = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; m < S; m += (uint64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < N; i++) {
            const double c = ((m >> i) & 1) ? c_w[i] : c_v[i];
            s += c * __ldg(x + (m ^ (1ull << i)));
        }
        out[m] = s;
    }
}

int main(int argc, char **argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 24;
    const int reps = argc > 2 ? atoi(argv[2]) : 10;
    const uint64_t S = 1ull << N;
    std::vector<uint32_t> binom(33 * 34, 0);
    for (int xx = 0; xx <= 32; xx++)
        for (int k = 0; k <= 33; k++) {
            double c = 1;
            if (k > xx) c = 0;
            else
                for (int t = 1; t <= k; t++) c = c * (xx - k + t) / t;
            binom[xx * 34 + k] = (uint32_t)llround(c);
        }
    std::vector<uint64_t> off(34, 0);
    for (int n = 0; n <= N; n++) off[n + 1] = off[n] + binom[N * 34 + n];
    double w[32], v[32];
    for (int i = 0; i < 32; i++) {
        w[i] = 0.3 + 0.01 * i;
        v[i] = 0.7 + 0.02 * i;
    }
    CK(cudaMemcpyToSymbol(c_w, w, sizeof(w)));
    CK(cudaMemcpyToSymbol(c_v, v, sizeof(v)));
    CK(cudaMemcpyToSymbol(c_off, off.data(), sizeof(uint64_t) * 34));
    CK(cudaMemcpyToSymbol(c_binom, binom.data(), sizeof(uint32_t) * 33 * 34));
    // natural x: x(m) = f(m); colex x: same values at their colex positions
    std::vector<double> xn(S), xc(S);
    std::vector<uint64_t> pos(S);
    for (uint64_t m = 0; m < S; m++) xn[m] = 1.0 + (double)((m * 2654435761ull) % 1000003ull) * 1e-6;
    {
        // colex order of each layer = increasing m among the sets of that size (colex = numeric
        // order of the bit pattern for equal popcount)
        std::vector<uint64_t> cnt(N + 1, 0);
        for (uint64_t m = 0; m < S; m++) {
            const int n = __builtin_popcountll(m);
            pos[m] = off[n] + cnt[n]++;
            xc[pos[m]] = xn[m];
        }
    }
    double *dxn, *dxc, *don, *doc;
    CK(cudaMalloc(&dxn, 8 * S));
    CK(cudaMalloc(&dxc, 8 * S));
    CK(cudaMalloc(&don, 8 * S));
    CK(cudaMalloc(&doc, 8 * S));
    CK(cudaMemcpy(dxn, xn.data(), 8 * S, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dxc, xc.data(), 8 * S, cudaMemcpyHostToDevice));
    constexpr int PER = 8;
    std::vector<uint64_t> tstart(N + 2, 0);
    for (int n = 0; n <= N; n++) tstart[n + 1] = tstart[n] + (binom[N * 34 + n] + PER - 1) / PER;
    uint64_t *dts;
    CK(cudaMalloc(&dts, 8 * (N + 2)));
    CK(cudaMemcpy(dts, tstart.data(), 8 * (N + 2), cudaMemcpyHostToDevice));
    const int tot = (int)tstart[N + 1];
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        std::vector<float> ts;
        for (int r = 0; r < reps; r++) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            ts.push_back(ms);
        }
        std::sort(ts.begin(), ts.end());
        return ts[ts.size() / 2];
    };
    const float tn = timeit([&] { k_natural2<<<nsm * 16, 256>>>(N, dxn, don); });
    const float tc = timeit([&] { k_colex<PER><<<(tot + 255) / 256, 256>>>(N, dxc, doc, dts, tot); });
    std::vector<double> on(S), oc(S);
    CK(cudaMemcpy(on.data(), don, 8 * S, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(oc.data(), doc, 8 * S, cudaMemcpyDeviceToHost));
    uint64_t bad = 0;
    for (uint64_t m = 0; m < S; m++)
        if (on[m] != oc[pos[m]]) bad++;
    const double alg = 16.0 * (double)S;   // compulsory: read x once, write out once
    printf("{\"N\": %d, \"states\": %llu, \"natural_ms\": %.4f, \"colex_ms\": %.4f, \"natural_ns_per_state\": %.4f, "
           "\"colex_ns_per_state\": %.4f, \"natural_compulsory_GBps\": %.1f, \"colex_compulsory_GBps\": %.1f, "
           "\"colex_over_natural\": %.3f, \"mismatches\": %llu}\n",
           N, (unsigned long long)S, tn, tc, 1e6 * tn / S, 1e6 * tc / S, alg / tn / 1e6, alg / tc / 1e6, tc / tn,
           (unsigned long long)bad);
    return bad ? 2 : 0;
}
