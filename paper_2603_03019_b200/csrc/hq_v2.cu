// hq_v2.cu -- the production sweep path (N >= 8) of the B200 solver.
//
// Design:
//  * Work unit = a warp tile of 128 parity-compressed states: compressed bits
//    0..4 are the lanes, bits 5..6 four register states per thread.  In the
//    internal unit order, units 0..7 vary inside a tile (unit 0 is the implied
//    parity bit, units 1..5 the lane bits, units 6..7 the register bits) and
//    units 8..N-1 are fixed by the tile index t (unit u <-> bit u-8 of t).
//  * Upward rates (Eq. tran_rates) never exist as a table.
//    Per tile a "rate program" is precomputed once per instance: for every
//    unit u the tile-uniform part W0_u = sum of Lambda_v over trie nodes of
//    unit u whose predecessor path is satisfied by the tile's fixed units and
//    uses no varying unit, plus a short list of (S, c) pairs, S = the varying
//    units the path needs.  W_u(m) = W0_u + sum_{S subset of m} c.  This is
//    Algorithm 3 evaluated symbolically for 128 states.
//  * Normalisation a priori: the closed-form inner fixed point of Algorithm 1
//    mu*(n) = (1 - sum_m b_m)/sum_m a_m (R1) is obtained BEFORE the
//    layer is touched from per-state scatter weights
//        omega(l) = sum_{i not in l} lambda_{l, l+i} / den(l+i),
//        kappa(l) = sum_{i in l}     nu_i              / den(l-i),
//    since sum_{m in C_n} a_m = sum_{l in C_{n-1}} p(l) omega(l) / lambda(n-1)
//    and sum_{m in C_n} b_m = lambda(n)/mu(n+1) sum_{l in C_{n+1}} p(l) kappa(l)
//    (exact reindexing of the sums in Eq. updateHeter).  So one pass per
//    half-sweep writes p_n(m) = (alpha_n A(m) + beta_n D(m)) / den(m) directly,
//    alpha_n = mu*(n)/lambda(n-1), beta_n = lambda(n)/mu(n+1).
//  * Tiles are visited in order of popcount(t) so that per-layer sums are kept
//    in 3 register bins per thread; the order also keeps the neighbour class
//    L2-resident up to N ~ 26.
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
// Precompute 3: per-tile rate programs.
// ---------------------------------------------------------------------------
struct PairAcc {
    int n;
    uint16_t key[PROG_MAXPAIRS];   // unit | S << 6
    double val[PROG_MAXPAIRS];
};

__device__ __forceinline__ bool pair_add(PairAcc &P, double *W0, int u, uint32_t S, double val) {
    if (S == 0) {
        W0[u] += val;
        return true;
    }
    const uint16_t key = (uint16_t)(u | (S << 6));
    for (int i = 0; i < P.n; i++)
        if (P.key[i] == key) {
            P.val[i] += val;
            return true;
        }
    if (P.n >= PROG_MAXPAIRS) return false;
    P.key[P.n] = key;
    P.val[P.n] = val;
    P.n++;
    return true;
}

// Walk the trie for tile t (fixed units 8.. given by F = t << 8).
__device__ bool tile_walk(const P2Args &a, uint32_t F, double *W0, PairAcc &P) {
    uint32_t Sst[HQ_MAXN + 2];
    Sst[0] = 0;
    for (int u = 0; u <= HQ_MAXN; u++) W0[u] = 0.0;
    P.n = 0;
    int v = 0;
    while (v < a.nnodes) {
        const int2 nd = __ldg(&a.node[v]);
        const int u = nd.x & 0xff;
        const int d = (nd.x >> 8) & 0xff;
        if (u >= PROG_NVARY && !((F >> u) & 1u)) {   // fixed and free: dead subtree
            v = nd.y;
            continue;
        }
        const uint32_t Spre = Sst[d - 1];
        const uint32_t Sme = Spre | (u < PROG_NVARY ? (1u << u) : 0u);
        // lane units (1..5) carry their own bit in the pattern, so that their
        // pairs only apply to lanes in which the unit is busy; units 0, 6, 7
        // get their own-busy condition from the register-state masks.
        const uint32_t Sp = (u >= 1 && u <= 5) ? Sme : Spre;
        if (!pair_add(P, W0, u, Sp, __ldg(&a.lam_thr[v]))) return false;
        if (!a.full_lists) {
            const double e = __ldg(&a.lam_end[v]);
            if (e != 0.0 && !pair_add(P, W0, a.N, Sme, e)) return false;
        }
        Sst[d] = Sme;
        v++;
    }
    return true;
}

__global__ void k_prog_count(P2Args a, const uint32_t *__restrict__ order, uint32_t *__restrict__ size16,
                             int *__restrict__ err) {
    PairAcc P;
    double W0[HQ_MAXN + 1];
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.ntiles;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = order[i];
        if (!tile_walk(a, t << 8, W0, P)) {
            atomicExch(err, 2);
            size16[i] = PROG_HDR16;
            continue;
        }
        int cnt[HQ_MAXN + 1];
        for (int u = 0; u <= HQ_MAXN; u++) cnt[u] = 0;
        for (int k = 0; k < P.n; k++) cnt[P.key[k] & 63]++;
        for (int u = 0; u <= HQ_MAXN; u++)
            if (cnt[u] > 32767) atomicExch(err, 3);
        size16[i] = PROG_HDR16 + (uint32_t)P.n;
    }
}

__global__ void k_prog_write(P2Args a, const uint32_t *__restrict__ order, const uint32_t *__restrict__ off16,
                             uint4 *__restrict__ prog) {
    PairAcc P;
    double W0[HQ_MAXN + 1];
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.ntiles;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = order[i];
        uint4 *out = prog + off16[i];
        if (!tile_walk(a, t << 8, W0, P)) continue;
        // stable sort of the pairs by (unit, class): class 0 = lane-only pattern
        // (no bit of units 0, 6, 7), class 1 = depends on the register state
        auto cls = [](uint16_t key) -> int { return (((key >> 6) & 0xC1u) != 0u) ? 1 : 0; };
        for (int x = 1; x < P.n; x++) {
            const uint16_t k = P.key[x];
            const double vv = P.val[x];
            const int kk = (k & 63) * 2 + cls(k);
            int y = x - 1;
            while (y >= 0 && ((P.key[y] & 63) * 2 + cls(P.key[y])) > kk) {
                P.key[y + 1] = P.key[y];
                P.val[y + 1] = P.val[y];
                y--;
            }
            P.key[y + 1] = k;
            P.val[y + 1] = vv;
        }
        uint32_t cw[32];
        for (int q = 0; q < 32; q++) cw[q] = 0;
        for (int k = 0; k < P.n; k++) {
            const int u = P.key[k] & 63;
            cw[u] += cls(P.key[k]) ? (1u << 16) : 1u;   // low half: lane-only count, high half: per-r count
        }
        for (int q = 0; q < 8; q++) out[q] = make_uint4(cw[4 * q], cw[4 * q + 1], cw[4 * q + 2], cw[4 * q + 3]);
        double *w0o = reinterpret_cast<double *>(out + PROG_CNT16);
        for (int u = 0; u < 32; u++) w0o[u] = u <= HQ_MAXN ? W0[u] : 0.0;
        for (int k = 0; k < P.n; k++) {
            const uint32_t S = P.key[k] >> 6;
            const int u = P.key[k] & 63;
            const uint32_t s0 = S & 1u, slane = (S >> 1) & 31u, sreg = (S >> 6) & 3u;
            uint32_t rm[2] = {0, 0};
            for (int beta = 0; beta < 2; beta++)
                for (int r = 0; r < 4; r++) {
                    const uint32_t b0 = (uint32_t)beta ^ (uint32_t)(__popc(r) & 1);
                    // own-busy condition of the register-state units (W_u is used only where u is busy)
                    const bool own = (u == 0) ? (b0 != 0) : (u == 6) ? ((r & 1) != 0) : (u == 7) ? ((r & 2) != 0) : true;
                    if ((sreg & ~(uint32_t)r) == 0 && (!s0 || b0) && own) rm[beta] |= 1u << r;
                }
            const uint32_t w = slane | (rm[0] << 8) | (rm[1] << 12) | ((uint32_t)u << 16);
            const double c = P.val[k];
            out[PROG_HDR16 + k] = make_uint4((uint32_t)__double_as_longlong(c),
                                             (uint32_t)(__double_as_longlong(c) >> 32), w, 0u);
        }
    }
}

// ---------------------------------------------------------------------------
// The sweep / residual kernel.
//   MODE 0: sweep (write p of the active layers of class c)
//   MODE 1: sweep + per-layer sum |p_new - p_old| (convergence proxy)
//   MODE 2: residual of Eq. balance_eq_heter for the states of class c
// NV per-layer values are reduced (sweep: p, p omega, p kappa [, p lambda]
// [, |dp|]; residual: |out - in|, out).
// ---------------------------------------------------------------------------
constexpr int WARPS = 8;

// acc += a * b if pred != 0 (forced predication: no selects, no branches)
__device__ __forceinline__ void pfma(double &acc, double a, double b, uint32_t pred) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\t@p fma.rn.f64 %0, %1, %2, %0;\n\t}"
        : "+d"(acc) : "d"(a), "d"(b), "r"(pred));
}

template <int NV>
__device__ __forceinline__ void flush_bins(double (&bins)[3][NV], int K, int c, int pcl, int lane,
                                           double (*wacc)[HQ_NV]) {
    if (K < 0) return;
    // bin k of this lane holds layer L_k = K + pcl + k + ((c ^ K ^ pcl ^ k) & 1)
    const int Lmin = K + ((c ^ K) & 1);
    int Lk[3];
#pragma unroll
    for (int k = 0; k < 3; k++) Lk[k] = K + pcl + k + ((c ^ K ^ pcl ^ k) & 1);
    for (int d = 0; d < 5; d++) {
        const int L = Lmin + 2 * d;
        if (L >= HQ_NL) break;
        const bool any = (Lk[0] == L) || (Lk[1] == L) || (Lk[2] == L);
        if (!__any_sync(0xffffffffu, any)) continue;
#pragma unroll
        for (int v = 0; v < NV; v++) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 3; k++) s += (Lk[k] == L) ? bins[k][v] : 0.0;
            s = warp_sum(s);
            if (lane == 0) wacc[L][v] += s;
        }
    }
#pragma unroll
    for (int k = 0; k < 3; k++)
#pragma unroll
        for (int v = 0; v < NV; v++) bins[k][v] = 0.0;
}

// lane-only pairs of one unit: Wt += c if the pattern's lane bits are busy in this lane
__device__ __forceinline__ double lane_pairs(const uint4 *__restrict__ my, int &pp, int cnt, uint32_t lane, double Wt) {
    for (int k = 0; k < cnt; k++) {
        const uint4 rec = __ldg(my + pp + k);
        const double cc = __hiloint2double((int)rec.y, (int)rec.x);
        const bool tl = ((rec.z & 31u) & ~lane) == 0u;
        Wt += tl ? cc : 0.0;
    }
    pp += cnt;
    return Wt;
}

// register-state pairs of one unit: A_r += c * q_r for the states r the pattern admits
__device__ __forceinline__ void reg_pairs(const uint4 *__restrict__ my, int &pp, int cnt, uint32_t lane, int beta,
                                          const double (&q)[4], double (&A)[4]) {
    const int sh = 8 + 4 * beta;
    for (int k = 0; k < cnt; k++) {
        const uint4 rec = __ldg(my + pp + k);
        const double cc = __hiloint2double((int)rec.y, (int)rec.x);
        const uint32_t w = rec.z;
        const uint32_t m4 = (((w & 31u) & ~lane) == 0u) ? ((w >> sh) & 15u) : 0u;
        pfma(A[0], cc, q[0], m4 & 1u);
        pfma(A[1], cc, q[1], m4 & 2u);
        pfma(A[2], cc, q[2], m4 & 4u);
        pfma(A[3], cc, q[3], m4 & 8u);
    }
    pp += cnt;
}

// uniform (REDUX) copy of a warp-uniform value: lets ptxas use uniform branches
__device__ __forceinline__ int wuni(int x) { return (int)__reduce_max_sync(0xffffffffu, (unsigned)x); }

// streaming load that does not allocate in L1 (L1 is kept for the rate programs)
__device__ __forceinline__ double ld_stream(const double *p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// prefetch the rate program of visit index i into L1 (one 128-byte line per lane)
__device__ __forceinline__ void prefetch_prog(const S2Args &a, uint64_t i, int lane) {
    if (i >= a.ntiles) return;
    const uint32_t o = __ldg(a.off16 + i);
    const uint32_t nrec = ((i + 1 < a.ntiles) ? __ldg(a.off16 + i + 1) : a.total16) - o;
    const char *base = reinterpret_cast<const char *>(a.prog + o);
    const uint32_t nlines = (nrec * 16 + 127) / 128 + 1;
    for (uint32_t k = lane; k < nlines; k += 32)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(base + 128 * (size_t)k));
}

// ---------------------------------------------------------------------------
// Per-warp TMA ring.  Every operand block of a tile (128 doubles = 1 KB:
// the own-index neighbours, the old p, the N-8 fixed-unit neighbour blocks,
// and the two halves of the scatter weights) is bulk-copied (cp.async.bulk,
// completion on an mbarrier) into a ring of RING slots; lanes 0..G-1 issue
// G blocks at once whenever G slots are free, so the copies run RING-G
// blocks ahead of the consumer without occupying registers.
// ---------------------------------------------------------------------------
constexpr int RING = 8;
constexpr int G = 4;

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void tma_load_1k(void *dst, const void *src, uint64_t *bar) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], 1024;" ::"r"(b) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 1024, [%2];"
                 ::"r"(d), "l"(src), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(b), "r"(parity) : "memory");
}

template <int MODE>
struct Stream {
    // block layout of one tile: [qown][pold?][nbr 8..N-1][omk lo, omk hi]?
    int nb;          // blocks per tile
    int nfix;        // N - 8
    __device__ __forceinline__ void init(int N) {
        nfix = N - PROG_NVARY;
        nb = 1 + (MODE >= 1 ? 1 : 0) + nfix + (MODE < 2 ? 2 : 0);
    }
    // source address of block b of the tile with index t
    __device__ __forceinline__ const void *src(const S2Args &a, uint32_t t, int b) const {
        const uint32_t jb = t << PROG_TB;
        int x = b;
        if (x == 0) return a.Q + jb;
        x--;
        if (MODE >= 1) {
            if (x == 0) return a.P + jb;
            x--;
        }
        if (x < nfix) return a.Q + (jb ^ (1u << (PROG_NVARY - 1 + x)));
        x -= nfix;
        return a.omkap + jb + 64 * x;
    }
};

template <int MODE, int NV, bool FULL>
__global__ void __launch_bounds__(WARPS * 32, 2) k_sweep2(S2Args a) {
    __shared__ double s_x[32];       // alpha(n) (sweep) or p(n-1) (residual)
    __shared__ double s_y[32];       // beta(n)  (sweep) or p(n+1)
    __shared__ double s_z[32];       // p(n) (residual)
    __shared__ double wacc[WARPS][HQ_NL][HQ_NV];
    __shared__ uint64_t sbar[WARPS][RING];
    extern __shared__ __align__(128) double sring[];   // [WARPS][RING][128]
    const int tid = threadIdx.x, lane = tid & 31, warp = wuni(threadIdx.x >> 5);
    for (int i = tid; i < WARPS * HQ_NL * HQ_NV; i += blockDim.x) (&wacc[0][0][0])[i] = 0.0;
    if (tid < 32) {
        if (MODE == 2) {
            const double *pn1 = a.coef + V2S_PN;   // pn1[n + 1] = p(n)
            s_x[tid] = pn1[tid];
            s_y[tid] = tid + 2 < 34 ? pn1[tid + 2] : 0.0;
            s_z[tid] = pn1[tid + 1];
        } else {
            s_x[tid] = a.coef[V2S_ALPHA + tid];
            s_y[tid] = a.coef[V2S_BETA + tid];
            s_z[tid] = 0.0;
        }
    }
    if (lane < RING) mbar_init(&sbar[warp][lane], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    double *__restrict__ ring = sring + (size_t)warp * RING * 128;
    uint64_t *bars = sbar[warp];

    const int pcl = __popc(lane);
    const uint64_t nwarps = (uint64_t)gridDim.x * WARPS;
    const uint64_t gw = (uint64_t)blockIdx.x * WARPS + warp;
    const uint64_t chunk = (a.ntiles + nwarps - 1) / nwarps;
    const uint64_t i0 = gw * chunk;
    const uint64_t i1 = min(i0 + chunk, a.ntiles);
    const int ntile_w = wuni(i1 > i0 ? (int)(i1 - i0) : 0);
    const uint32_t fullm = (1u << a.N) - 1u;
    const uint32_t ulane = (uint32_t)lane;

    Stream<MODE> st;
    st.init(a.N);
    const int total_blocks = ntile_w * st.nb;
    int issued = 0, consumed = 0;
    // issue blocks [issued, min(upto, total)) in batches: lane l issues block issued + l
    auto produce = [&](int upto) {
        upto = min(upto, total_blocks);
        while (issued + G <= upto || (issued < upto && upto == total_blocks)) {
            const int nbatch = min(G, upto - issued);
            if (lane < nbatch) {
                const int gb = issued + lane;
                const int tt = gb / st.nb, b = gb - tt * st.nb;
                const uint32_t tix = __ldg(a.order + i0 + tt);
                const int slot = gb % RING;
                tma_load_1k(ring + slot * 128, st.src(a, tix, b), &bars[slot]);
            }
            issued += nbatch;
        }
    };
    // wait for the next block, copy it to registers, release the slot
    auto consume4 = [&](double (&v)[4]) {
        const int slot = consumed % RING;
        mbar_wait(&bars[slot], (unsigned)((consumed / RING) & 1));
        const double *blk = ring + slot * 128;
#pragma unroll
        for (int r = 0; r < 4; r++) v[r] = blk[r * 32 + lane];
        __syncwarp();
        consumed++;
        produce(consumed + RING);
    };
    auto consume_ok = [&](double2 (&v)[4]) {   // two blocks of 64 double2: r = 0,1 then r = 2,3
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int slot = consumed % RING;
            mbar_wait(&bars[slot], (unsigned)((consumed / RING) & 1));
            const double2 *blk = reinterpret_cast<const double2 *>(ring + slot * 128);
            v[2 * h] = blk[lane];
            v[2 * h + 1] = blk[32 + lane];
            __syncwarp();
            consumed++;
            produce(consumed + RING);
        }
    };

    double mu_lane = 0.0;
#pragma unroll
    for (int b = 0; b < 5; b++)
        if ((lane >> b) & 1) mu_lane += a.nu[1 + b];

    double bins[3][NV];
#pragma unroll
    for (int k = 0; k < 3; k++)
#pragma unroll
        for (int v = 0; v < NV; v++) bins[k][v] = 0.0;
    int curK = -1;
    produce(RING);
    if (ntile_w > 0) prefetch_prog(a, i0, lane);

    for (int it = 0; it < ntile_w; it++) {
        const uint64_t i = i0 + it;
        const uint32_t t = (uint32_t)wuni((int)__ldg(a.order + i));
        const int K = __popc(t);
        const uint32_t jb = t << PROG_TB;
        if (it + 1 < ntile_w) prefetch_prog(a, i + 1, lane);
        if (K != curK) {
            flush_bins<NV>(bins, curK, a.c, pcl, lane, wacc[warp]);
            curK = K;
        }
        double qo[4];
        consume4(qo);
        double pold[4];
        if (MODE >= 1) consume4(pold);
        const uint4 *__restrict__ my = a.prog + __ldg(a.off16 + i);
        const uint32_t *__restrict__ mycnt = reinterpret_cast<const uint32_t *>(my);
        const double *__restrict__ myw0 = reinterpret_cast<const double *>(my + PROG_CNT16);
        const int beta = (a.c ^ K ^ pcl) & 1;
        int pp = PROG_HDR16;
        double A[4] = {0.0, 0.0, 0.0, 0.0}, D[4] = {0.0, 0.0, 0.0, 0.0};
        double mu_fix = 0.0;
        // ---- unit 0 (implied parity bit): busy in r iff b0(r) = beta ^ parity(r)
        {
            const uint32_t cw = (uint32_t)wuni((int)__ldg(mycnt + 0));
            const double Wt = lane_pairs(my, pp, (int)(cw & 0xffffu), ulane, __ldg(myw0 + 0));
            const double nu = a.nu[0];
            const double We = beta ? Wt : 0.0, Wo = beta ? 0.0 : Wt;   // r = 0,3 / r = 1,2
            const double ne = beta ? 0.0 : nu, no = beta ? nu : 0.0;
            A[0] = fma(We, qo[0], A[0]);
            A[3] = fma(We, qo[3], A[3]);
            A[1] = fma(Wo, qo[1], A[1]);
            A[2] = fma(Wo, qo[2], A[2]);
            D[0] = fma(ne, qo[0], D[0]);
            D[3] = fma(ne, qo[3], D[3]);
            D[1] = fma(no, qo[1], D[1]);
            D[2] = fma(no, qo[2], D[2]);
            reg_pairs(my, pp, (int)(cw >> 16), ulane, beta, qo, A);
        }
        // ---- lane units 1..5: busy per lane; own lane bit is part of every pattern
#pragma unroll
        for (int u = 1; u <= 5; u++) {
            double q[4];
#pragma unroll
            for (int r = 0; r < 4; r++) q[r] = __shfl_xor_sync(0xffffffffu, qo[r], 1 << (u - 1));
            const uint32_t cw = (uint32_t)wuni((int)__ldg(mycnt + u));
            const double Wt = lane_pairs(my, pp, (int)(cw & 0xffffu), ulane, 0.0);
            const double nut = ((lane >> (u - 1)) & 1) ? 0.0 : a.nu[u];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                A[r] = fma(Wt, q[r], A[r]);
                D[r] = fma(nut, q[r], D[r]);
            }
            reg_pairs(my, pp, (int)(cw >> 16), ulane, beta, q, A);
        }
        // ---- register units 6, 7: busy in the register states with the bit set
#pragma unroll
        for (int u = 6; u <= 7; u++) {
            const int bit = 1 << (u - 6);
            double q[4];
#pragma unroll
            for (int r = 0; r < 4; r++) q[r] = qo[r ^ bit];
            const uint32_t cw = (uint32_t)wuni((int)__ldg(mycnt + u));
            const double Wt = lane_pairs(my, pp, (int)(cw & 0xffffu), ulane, __ldg(myw0 + u));
            const double nu = a.nu[u];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                if (r & bit) A[r] = fma(Wt, q[r], A[r]);
                else D[r] = fma(nu, q[r], D[r]);
            }
            reg_pairs(my, pp, (int)(cw >> 16), ulane, beta, q, A);
        }
        // ---- fixed units 8..N-1 (tile-uniform busy status), neighbour blocks from the ring
        for (int u = PROG_NVARY; u < a.N; u++) {
            double q[4];
            consume4(q);
            const double nu = a.nu[u];
            if (!((t >> (u - PROG_NVARY)) & 1u)) {
#pragma unroll
                for (int r = 0; r < 4; r++) D[r] = fma(nu, q[r], D[r]);
                continue;
            }
            mu_fix += nu;
            const uint32_t cw = (uint32_t)wuni((int)__ldg(mycnt + u));
            const double Wt = lane_pairs(my, pp, (int)(cw & 0xffffu), ulane, __ldg(myw0 + u));
#pragma unroll
            for (int r = 0; r < 4; r++) A[r] = fma(Wt, q[r], A[r]);
            reg_pairs(my, pp, (int)(cw >> 16), ulane, beta, q, A);
        }
        // ---- lambda_m (blocked pseudo-unit for truncated lists)
        double lam[4];
        if (FULL) {
#pragma unroll
            for (int r = 0; r < 4; r++) lam[r] = a.Lam;
        } else {
            const int u = a.N;
            const uint32_t cw = (uint32_t)wuni((int)__ldg(mycnt + u));
            const double Bt = lane_pairs(my, pp, (int)(cw & 0xffffu), ulane, __ldg(myw0 + u));
            double Bk[4] = {Bt, Bt, Bt, Bt};
            const double one[4] = {1.0, 1.0, 1.0, 1.0};
            reg_pairs(my, pp, (int)(cw >> 16), ulane, beta, one, Bk);
#pragma unroll
            for (int r = 0; r < 4; r++) lam[r] = a.Lam - Bk[r];
        }
        double2 okv[4];
        if (MODE < 2) consume_ok(okv);
#pragma unroll
        for (int r = 0; r < 4; r++) {
            const int pr = __popc(r);
            const int b0r = beta ^ (pr & 1);
            const int n = K + pcl + pr + b0r;
            const uint32_t j = jb + r * 32 + lane;
            const double mu = mu_fix + mu_lane + (b0r ? a.nu[0] : 0.0) + ((r & 1) ? a.nu[6] : 0.0) +
                              ((r & 2) ? a.nu[7] : 0.0);
            double lm = lam[r];
            if (FULL && (((j << 1) | (uint32_t)b0r) == fullm)) lm = 0.0;
            const double den = lm + mu;
            if (MODE == 2) {
                const double out = s_z[n] * pold[r] * den;
                const double in = s_x[n] * A[r] + s_y[n] * D[r];
                bins[pr][0] += fabs(out - in);
                bins[pr][1] += out;
            } else {
                if (!((a.active >> n) & 1u)) continue;
                const double rden = __drcp_rn(den);
                const double p = (s_x[n] * A[r] + s_y[n] * D[r]) * rden;
                a.P[j] = p;
                const double2 ok = okv[r];
                bins[pr][0] += p;
                bins[pr][1] += p * ok.x;
                bins[pr][2] += p * ok.y;
                if (!FULL) bins[pr][3] += p * lm;
                if (MODE == 1) bins[pr][NV - 1] += fabs(p - pold[r]);
            }
        }
    }
    flush_bins<NV>(bins, curK, a.c, pcl, lane, wacc[warp]);
    __syncthreads();
    double *out = a.partial + (size_t)blockIdx.x * HQ_NL * HQ_NV;
    for (int i = tid; i < HQ_NL * HQ_NV; i += blockDim.x) {
        const int L = i / HQ_NV, v = i % HQ_NV;
        double s = 0.0;
        int src = -1;
        if (MODE == 2) src = (v < 2) ? v : -1;
        else if (v == V2_P) src = 0;
        else if (v == V2_OM) src = 1;
        else if (v == V2_KA) src = 2;
        else if (v == V2_LAM) src = FULL ? -1 : 3;
        else if (v == V2_DL1) src = (MODE == 1) ? NV - 1 : -1;
        if (src >= 0) {
#pragma unroll
            for (int w = 0; w < WARPS; w++) s += wacc[w][L][src];
        }
        out[L * HQ_NV + v] = s;
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
cudaError_t prog_count(const P2Args &a, const uint32_t *order, uint32_t *size16, int *err, int grid, cudaStream_t s) {
    hq2::k_prog_count<<<grid, 128, 0, s>>>(a, order, size16, err);
    return cudaGetLastError();
}
cudaError_t prog_scan(const uint32_t *size16, uint32_t *off16, uint64_t n, void *tmp, size_t *tmp_bytes,
                      cudaStream_t s) {
    return cub::DeviceScan::ExclusiveSum(tmp, *tmp_bytes, size16, off16, (int)n, s);
}
cudaError_t prog_write(const P2Args &a, const uint32_t *order, const uint32_t *off16, uint4 *prog, int grid,
                       cudaStream_t s) {
    hq2::k_prog_write<<<grid, 128, 0, s>>>(a, order, off16, prog);
    return cudaGetLastError();
}
size_t sweep_smem(uint32_t maxrec) { (void)maxrec; return sizeof(double) * 128 * hq2::RING * hq2::WARPS; }

template <int MODE, int NV, bool FULL>
static cudaError_t launch_sweep(const S2Args &a, int grid, cudaStream_t s) {
    const size_t sm = sweep_smem(a.maxrec);
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(hq2::k_sweep2<MODE, NV, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        attr_set = true;
    }
    hq2::k_sweep2<MODE, NV, FULL><<<grid, hq2::WARPS * 32, sm, s>>>(a);
    return cudaGetLastError();
}

cudaError_t sweep(const S2Args &a, int mode, int grid, cudaStream_t s) {
    if (a.full_lists) {
        if (mode == 0) return launch_sweep<0, 3, true>(a, grid, s);
        if (mode == 1) return launch_sweep<1, 4, true>(a, grid, s);
        return launch_sweep<2, 2, true>(a, grid, s);
    }
    if (mode == 0) return launch_sweep<0, 4, false>(a, grid, s);
    if (mode == 1) return launch_sweep<1, 5, false>(a, grid, s);
    return launch_sweep<2, 2, false>(a, grid, s);
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
