// hq_v3.cu -- CTA-tiled sweep kernel of the B200 solver (N >= 9).
//
// One half-sweep of the red-black staggered Algorithm 1 (
// DESIGN.md §2) updates every state m of parity class c:
//     p_n(m) = (alpha_n A(m) + beta_n D(m)) / (lambda_m + mu_m)          (Eq. updateHeter)
//     A(m)   = sum_{i busy}  W_i(m) q(m - i),  W_i(m) = lambda_{m-i -> m} (Eq. tran_rates)
//     D(m)   = sum_{i free}  nu_i   q(m + i)
// with q = the other class and alpha_n = mu*(n)/lambda(n-1), beta_n =
// lambda(n)/mu(n+1) prepared a priori (hq_v2.cu k_scalars2, R1).
//
// Work decomposition (hq_v3.h): a CTA of 32 << nW threads owns one tile of
// 2^T compressed states (T = 8 + nW) at a time.  Thread (w, l) owns 8 states.
// Neighbours across
//   * register bits (units 1, 7, 8) come from the thread's own registers,
//   * the implied parity unit 0 is the state's own index in the other class,
//   * lane and warp bits (units 2..6, 9..8+nW) come from the tile's block of q
//     staged in shared memory by one bulk copy (TMA engine, cp.async.bulk),
//   * tile bits ("H" units) come from the neighbour tile's block, streamed per
//     warp through a 4-slot ring of 2 KB bulk copies completed on mbarriers.
// The upward rates are evaluated from a per-tile "rate program"
// (Algorithm 3, evaluated symbolically for the 2^T states
// of the tile): per unit a tile-uniform part W0_u plus pairs (c, S) added when
// the varying units S are busy.  Pairs that depend only on lane/warp units
// are summed once per thread; pairs that involve register units or the
// parity unit carry an 8-bit mask of the admissible register states.
//
// Per-layer sums (sum p, sum p omega, sum p kappa [, sum p lambda_m]
// [, sum |dp|]) are accumulated in fixed order: per-thread bins, warp
// butterflies keyed by layer when popcount(tile) changes, a fixed-order sum
// over the warps of the CTA, and k_scalars2's fixed-order sum over CTAs.
#include <cuda_runtime.h>
#include <cstdint>
#include "hq_internal.h"
#include "hq_v2.h"
#include "hq_v3.h"

namespace hq3 {

constexpr int R = V3_R;
constexpr int RING = V3_RING;

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}
__device__ __forceinline__ int wuni(int x) { return (int)__reduce_max_sync(0xffffffffu, (unsigned)x); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(b),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// acc += a * b if pred != 0 (forced predication)
__device__ __forceinline__ void pfma(double &acc, double a, double b, uint32_t pred) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\t@p fma.rn.f64 %0, %1, %2, %0;\n\t}"
        : "+d"(acc)
        : "d"(a), "d"(b), "r"(pred));
}

__device__ __forceinline__ double rec_c(const uint4 &x) { return __hiloint2double((int)x.y, (int)x.x); }

// tile-uniform part plus the lane-only pairs whose thread-level condition holds
__device__ __forceinline__ double lane_pairs(const uint4 *__restrict__ rec, int n, uint32_t busy_t, double W) {
    for (int k = 0; k < n; k++) {
        const uint4 x = rec[k];
        if ((x.z & ~busy_t) == 0u) W += rec_c(x);
    }
    return W;
}

// register-dependent pairs: A[r] += c q[r] for the admissible states r
__device__ __forceinline__ void reg_pairs(const uint4 *__restrict__ rec, int n, uint32_t busy_t, int sh,
                                          const double (&q)[R], double (&A)[R]) {
    for (int k = 0; k < n; k++) {
        const uint4 x = rec[k];
        const double c = rec_c(x);
        const uint32_t m8 = ((x.z & ~busy_t) == 0u) ? ((x.w >> sh) & 0xffu) : 0u;
#pragma unroll
        for (int r = 0; r < R; r++) pfma(A[r], c, q[r], m8 & (1u << r));
    }
}

// value slots (partial[..][layer][slot]) of the reduced quantities
template <int MODE, bool FULL>
struct Slots {
    static constexpr int NB = MODE == 2 ? 2 : 3 + (FULL ? 0 : 1) + (MODE == 1 ? 1 : 0);
    __device__ static constexpr int slot(int v) {
        return MODE == 2 ? v : (v < 3 ? v : (!FULL && v == 3) ? V2_LAM : V2_DL1);
    }
};

template <int MODE, bool FULL>
__global__ void __launch_bounds__(512, 1) k_sweep3(S3Args a) {
    using SL = Slots<MODE, FULL>;
    constexpr int NB = SL::NB;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t tbar[2];
    __shared__ __align__(8) uint64_t rbar[16][RING];
    __shared__ double s_x[32], s_y[32], s_z[32], s_mr[R];

    const int nW = a.nW, T = 8 + nW, NVU = 9 + nW, nH = a.N - NVU;
    const int tid = threadIdx.x, lane = tid & 31, warp = wuni(tid >> 5);
    const uint32_t tstates = 1u << T;
    double *tileq = reinterpret_cast<double *>(smem_raw);
    uint4 *progb = reinterpret_cast<uint4 *>(tileq + 2 * tstates);
    double *ring = reinterpret_cast<double *>(progb + 2 * a.maxrec16) + (size_t)warp * RING * V3_SLOT;

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
        if (tid < R)
            s_mr[tid] = ((tid & 1) ? a.nu[1] : 0.0) + ((tid & 2) ? a.nu[7] : 0.0) + ((tid & 4) ? a.nu[8] : 0.0);
    }
    if (tid == 0) {
        mbar_init(&tbar[0], 1);
        mbar_init(&tbar[1], 1);
    }
    if (lane < RING) mbar_init(&rbar[warp][lane], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();

    const uint64_t i0 = (uint64_t)blockIdx.x * a.chunk;
    const uint64_t i1 = min(i0 + a.chunk, a.ntiles);
    const int nt = i1 > i0 ? (int)(i1 - i0) : 0;

    // ---- CTA-level tile loader (thread 0): q block of the tile + its rate program
    auto load_tile = [&](int k) {
        const uint64_t idx = i0 + k;
        const uint32_t t = __ldg(a.order + idx);
        const uint32_t o = __ldg(a.off16 + idx);
        const uint32_t nrec = (idx + 1 < a.ntiles ? __ldg(a.off16 + idx + 1) : a.total16) - o;
        const int buf = k & 1;
        mbar_expect(&tbar[buf], tstates * 8u + nrec * 16u);
        bulk_g2s(tileq + (size_t)buf * tstates, a.Q + ((size_t)t << T), tstates * 8u, &tbar[buf]);
        bulk_g2s(progb + (size_t)buf * a.maxrec16, a.prog + o, nrec * 16u, &tbar[buf]);
    };

    // ---- per-warp ring: items of a tile = H-unit neighbour slices [, own p] [, omega/kappa x 2]
    const int nitems = nH + (MODE >= 1 ? 1 : 0) + (MODE < 2 ? 2 : 0);
    const int total = nt * nitems;
    int issued = 0, consumed = 0, pk = 0, pb = 0;
    uint32_t pt = nt > 0 ? __ldg(a.order + i0) : 0u;
    const uint32_t wb = (uint32_t)warp << 8;
    auto issue_next = [&]() {
        if (lane == 0) {
            const uint32_t jt = pt << T;
            const void *src;
            if (pb < nH) src = a.Q + ((jt ^ (1u << (T + pb))) + wb);
            else if (MODE >= 1 && pb == nH) src = a.P + (jt + wb);
            else src = a.omkap + (jt + wb) + 128u * (uint32_t)(pb - nH - (MODE >= 1 ? 1 : 0));
            const int slot = issued & (RING - 1);
            fence_proxy_async();
            mbar_expect(&rbar[warp][slot], V3_SLOT * 8u);
            bulk_g2s(ring + slot * V3_SLOT, src, V3_SLOT * 8u, &rbar[warp][slot]);
        }
        issued++;
        if (++pb == nitems) {
            pb = 0;
            if (++pk < nt) pt = __ldg(a.order + i0 + pk);
        }
    };
    auto produce = [&]() {
        while (issued < total && issued < consumed + RING) issue_next();
    };
    auto wait_at = [&](int ahead) -> const double * {   // item consumed + ahead
        const int g = consumed + ahead;
        const int slot = g & (RING - 1);
        mbar_wait(&rbar[warp][slot], (unsigned)((g / RING) & 1));
        return ring + slot * V3_SLOT;
    };
    auto wait_slot = [&]() -> const double * { return wait_at(0); };
    auto release_n = [&](int n) {
        __syncwarp();
        consumed += n;
        produce();
    };
    auto release = [&]() { release_n(1); };

    produce();
    if (tid == 0 && nt > 0) load_tile(0);

    // ---- per-thread constants
    const uint32_t busy_t = ((uint32_t)lane << 2) | ((uint32_t)warp << 9);   // L units 2..6, W units 9..
    double mu_t = 0.0;
#pragma unroll
    for (int b = 0; b < 5; b++)
        if ((lane >> b) & 1) mu_t += a.nu[2 + b];
    for (int b = 0; b < nW; b++)
        if ((warp >> b) & 1) mu_t += a.nu[9 + b];
    const int popc_t = __popc(lane) + __popc(warp);
    const int par_t = popc_t & 1;
    const uint32_t jw = ((uint32_t)warp << 8) | ((uint32_t)lane << 1);   // j_local(r) = jw | (r>>1)<<6 | (r&1)
    const double nu0 = a.nu[0];

    double acc[NB];   // lane L: layer L
#pragma unroll
    for (int v = 0; v < NB; v++) acc[v] = 0.0;
    double bins[3][NB];
#pragma unroll
    for (int h = 0; h < 3; h++)
#pragma unroll
        for (int v = 0; v < NB; v++) bins[h][v] = 0.0;
    int curK = -1;

    auto flush = [&]() {
        if (curK < 0) return;
        const int betaK = a.c ^ (curK & 1) ^ par_t;
        const int Lb = curK + popc_t + betaK;   // layers Lb, Lb + 2, Lb + 4
        const int L0 = curK + __popc(warp);
        for (int Lc = L0; Lc <= L0 + 10 && Lc < HQ_NL; Lc++) {
            if ((Lc & 1) != a.c) continue;
            const bool any = (Lb == Lc) || (Lb + 2 == Lc) || (Lb + 4 == Lc);
            if (!__any_sync(0xffffffffu, any)) continue;
#pragma unroll
            for (int v = 0; v < NB; v++) {
                double s = (Lb == Lc ? bins[0][v] : 0.0) + (Lb + 2 == Lc ? bins[1][v] : 0.0) +
                           (Lb + 4 == Lc ? bins[2][v] : 0.0);
                s = warp_sum(s);
                if (lane == Lc) acc[v] += s;
            }
        }
#pragma unroll
        for (int h = 0; h < 3; h++)
#pragma unroll
            for (int v = 0; v < NB; v++) bins[h][v] = 0.0;
    };

    for (int k = 0; k < nt; k++) {
        const int buf = k & 1;
        const uint32_t t = (uint32_t)wuni((int)__ldg(a.order + i0 + k));
        mbar_wait(&tbar[buf], (unsigned)((k >> 1) & 1));
        __syncthreads();   // every warp is done with tile k-1: its buffer may be refilled
        if (tid == 0 && k + 1 < nt) {
            fence_proxy_async();
            load_tile(k + 1);
        }
        const double *tq = tileq + (size_t)buf * tstates;
        const uint4 *pg = progb + (size_t)buf * a.maxrec16;
        const uint32_t *info = reinterpret_cast<const uint32_t *>(pg);
        const double *W0 = reinterpret_cast<const double *>(pg + 8);
        const uint4 *pr = pg + V3_HDR16;
        const int K = __popc(t);
        if (K != curK) {
            flush();
            curK = K;
        }
        const int beta = a.c ^ (K & 1) ^ par_t;
        const int sh = beta ? 8 : 0;
        double mu_F = 0.0;
        for (int h = 0; h < nH; h++)
            if ((t >> h) & 1u) mu_F += a.nu[NVU + h];

        double qo[R], A[R], D[R], q[R];
#pragma unroll
        for (int kk = 0; kk < 4; kk++) {
            const double2 v = *reinterpret_cast<const double2 *>(tq + (jw | (kk << 6)));
            qo[2 * kk] = v.x;
            qo[2 * kk + 1] = v.y;
        }
#pragma unroll
        for (int r = 0; r < R; r++) {
            A[r] = 0.0;
            D[r] = 0.0;
        }
        // ---- unit 0 (implied parity bit): busy in r iff b0(r) = beta ^ parity(r)
        {
            const uint32_t inf = info[0];
            const uint4 *p0 = pr + (inf >> 16);
            const double Wt = lane_pairs(p0, (int)(inf & 0xffu), busy_t, W0[0]);
            const double We = beta ? Wt : 0.0, Wo = beta ? 0.0 : Wt;
            const double Ne = beta ? 0.0 : nu0, No = beta ? nu0 : 0.0;
#pragma unroll
            for (int r = 0; r < R; r++) {
                const bool odd = (__popc(r) & 1) != 0;
                A[r] = fma(odd ? Wo : We, qo[r], A[r]);
                D[r] = fma(odd ? No : Ne, qo[r], D[r]);
            }
            reg_pairs(p0 + (inf & 0xffu), (int)((inf >> 8) & 0xffu), busy_t, sh, qo, A);
        }
        // ---- register units 1, 7, 8 (register bits 0, 1, 2)
#pragma unroll
        for (int rb = 0; rb < 3; rb++) {
            const int u = rb ? 6 + rb : 1;
            const int bit = 1 << rb;
            const uint32_t inf = info[u];
            const uint4 *p0 = pr + (inf >> 16);
            const double Wt = lane_pairs(p0, (int)(inf & 0xffu), busy_t, W0[u]);
            const double nuu = a.nu[u];
#pragma unroll
            for (int r = 0; r < R; r++) q[r] = qo[r ^ bit];
#pragma unroll
            for (int r = 0; r < R; r++) {
                if (r & bit) A[r] = fma(Wt, q[r], A[r]);
                else D[r] = fma(nuu, q[r], D[r]);
            }
            reg_pairs(p0 + (inf & 0xffu), (int)((inf >> 8) & 0xffu), busy_t, sh, q, A);
        }
        // ---- lane units 2..6 (lane bits 0..4): busy per lane
#pragma unroll
        for (int b = 0; b < 5; b++) {
            const int u = 2 + b;
            const uint32_t inf = info[u];
            const uint4 *p0 = pr + (inf >> 16);
            const bool busy = (lane >> b) & 1;
            const uint32_t jn = jw ^ (2u << b);
#pragma unroll
            for (int kk = 0; kk < 4; kk++) {
                const double2 v = *reinterpret_cast<const double2 *>(tq + (jn | (kk << 6)));
                q[2 * kk] = v.x;
                q[2 * kk + 1] = v.y;
            }
            // the pairs of a lane unit carry its own bit: they vanish where it is free
            const double Wt = lane_pairs(p0, (int)(inf & 0xffu), busy_t, busy ? W0[u] : 0.0);
            const double wn = busy ? 0.0 : a.nu[u];
#pragma unroll
            for (int r = 0; r < R; r++) {
                A[r] = fma(Wt, q[r], A[r]);
                D[r] = fma(wn, q[r], D[r]);
            }
            reg_pairs(p0 + (inf & 0xffu), (int)((inf >> 8) & 0xffu), busy_t, sh, q, A);
        }
        // ---- warp units 9..8+nW (warp bits): busy per warp (uniform branch)
        for (int b = 0; b < nW; b++) {
            const int u = 9 + b;
            const uint32_t jn = jw ^ (256u << b);
#pragma unroll
            for (int kk = 0; kk < 4; kk++) {
                const double2 v = *reinterpret_cast<const double2 *>(tq + (jn | (kk << 6)));
                q[2 * kk] = v.x;
                q[2 * kk + 1] = v.y;
            }
            if ((warp >> b) & 1) {
                const uint32_t inf = info[u];
                const uint4 *p0 = pr + (inf >> 16);
                const double Wt = lane_pairs(p0, (int)(inf & 0xffu), busy_t, W0[u]);
#pragma unroll
                for (int r = 0; r < R; r++) A[r] = fma(Wt, q[r], A[r]);
                reg_pairs(p0 + (inf & 0xffu), (int)((inf >> 8) & 0xffu), busy_t, sh, q, A);
            } else {
                const double nuu = a.nu[u];
#pragma unroll
                for (int r = 0; r < R; r++) D[r] = fma(nuu, q[r], D[r]);
            }
        }
        // ---- tile units (H): neighbour tile slices from the ring, busy per tile
        for (int h = 0; h < nH; h++) {
            const int u = NVU + h;
            const double *sl = wait_slot();
#pragma unroll
            for (int kk = 0; kk < 4; kk++) {
                const double2 v = *reinterpret_cast<const double2 *>(sl + ((lane << 1) | (kk << 6)));
                q[2 * kk] = v.x;
                q[2 * kk + 1] = v.y;
            }
            release();
            if ((t >> h) & 1u) {
                const uint32_t inf = info[u];
                const uint4 *p0 = pr + (inf >> 16);
                const double Wt = lane_pairs(p0, (int)(inf & 0xffu), busy_t, W0[u]);
#pragma unroll
                for (int r = 0; r < R; r++) A[r] = fma(Wt, q[r], A[r]);
                reg_pairs(p0 + (inf & 0xffu), (int)((inf >> 8) & 0xffu), busy_t, sh, q, A);
            } else {
                const double nuu = a.nu[u];
#pragma unroll
                for (int r = 0; r < R; r++) D[r] = fma(nuu, q[r], D[r]);
            }
        }
        // ---- own old p (convergence proxy / residual): read in the epilogue, slot held until then
        const double *slp = MODE >= 1 ? wait_at(0) : nullptr;
        // ---- lambda_m: Lambda minus the atoms whose whole (truncated) list is busy
        double lam[R];
        if (FULL) {
#pragma unroll
            for (int r = 0; r < R; r++) lam[r] = a.Lam;
        } else {
            const int u = a.N;
            const uint32_t inf = info[u];
            const uint4 *p0 = pr + (inf >> 16);
            const double Bt = lane_pairs(p0, (int)(inf & 0xffu), busy_t, W0[u]);
            double one[R];
#pragma unroll
            for (int r = 0; r < R; r++) {
                lam[r] = Bt;
                one[r] = 1.0;
            }
            reg_pairs(p0 + (inf & 0xffu), (int)((inf >> 8) & 0xffu), busy_t, sh, one, lam);
#pragma unroll
            for (int r = 0; r < R; r++) lam[r] = a.Lam - lam[r];
        }
        // ---- scatter weights omega, kappa of the updated states (two slots, read in the epilogue)
        const double2 *slo0 = nullptr, *slo1 = nullptr;
        if (MODE < 2) {
            const int o = MODE >= 1 ? 1 : 0;
            slo0 = reinterpret_cast<const double2 *>(wait_at(o));
            slo1 = reinterpret_cast<const double2 *>(wait_at(o + 1));
        }
        // ---- epilogue
        const int base = K + popc_t;
        const double mu_base = mu_F + mu_t;
        const uint32_t jt = t << T;
        double pnew[R];
        bool act[R];
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int pc = __popc(r);
            const int b0 = beta ^ (pc & 1);
            const int n = base + pc + b0;
            const double mu = mu_base + s_mr[r] + (b0 ? nu0 : 0.0);
            double lm = lam[r];
            if (FULL && n == a.N) lm = 0.0;
            const double den = lm + mu;
            double val[NB];
            act[r] = true;
            const int so = ((r >> 1) << 6) | (lane << 1) | (r & 1);   // warp-local state offset
            const double pold = MODE >= 1 ? slp[so] : 0.0;
            if (MODE == 2) {
                const double out = s_z[n] * pold * den;
                const double in = s_x[n] * A[r] + s_y[n] * D[r];
                val[0] = fabs(out - in);
                val[1] = out;
            } else {
                act[r] = (a.active >> n) & 1u;
                const double p = (s_x[n] * A[r] + s_y[n] * D[r]) * __drcp_rn(den);
                const double2 ok = (r < 4 ? slo0 : slo1)[so & 127];
                pnew[r] = p;
                val[0] = act[r] ? p : 0.0;
                val[1] = act[r] ? p * ok.x : 0.0;
                val[2] = act[r] ? p * ok.y : 0.0;
                int v = 3;
                if (!FULL) val[v++] = act[r] ? p * lm : 0.0;
                if (MODE == 1) val[v++] = act[r] ? fabs(p - pold) : 0.0;
            }
            // bin h(r) = (pc + 1 - beta) >> 1
#pragma unroll
            for (int v = 0; v < NB; v++) {
                if (pc == 0) bins[0][v] += val[v];
                else if (pc == 2) bins[1][v] += val[v];
                else if (pc == 1) {
                    if (beta) bins[0][v] += val[v];
                    else bins[1][v] += val[v];
                } else {
                    if (beta) bins[1][v] += val[v];
                    else bins[2][v] += val[v];
                }
            }
        }
        release_n((MODE >= 1 ? 1 : 0) + (MODE < 2 ? 2 : 0));
        if (MODE < 2) {
#pragma unroll
            for (int kk = 0; kk < 4; kk++) {
                double *dst = a.P + (jt + (jw | (kk << 6)));
                if (act[2 * kk] && act[2 * kk + 1]) {
                    *reinterpret_cast<double2 *>(dst) = make_double2(pnew[2 * kk], pnew[2 * kk + 1]);
                } else {
                    if (act[2 * kk]) dst[0] = pnew[2 * kk];
                    if (act[2 * kk + 1]) dst[1] = pnew[2 * kk + 1];
                }
            }
        }
    }
    flush();
    // ---- CTA partials: warp w's lane L holds layer L; fixed-order sum over warps
    __syncwarp();
#pragma unroll
    for (int v = 0; v < NB; v++) ring[lane * NB + v] = acc[v];
    __syncthreads();
    if (warp == 0) {
        const double *base = reinterpret_cast<const double *>(progb + 2 * a.maxrec16);
        double s[NB];
#pragma unroll
        for (int v = 0; v < NB; v++) s[v] = 0.0;
        for (int w = 0; w < (1 << nW); w++)
#pragma unroll
            for (int v = 0; v < NB; v++) s[v] += base[(size_t)w * RING * V3_SLOT + lane * NB + v];
        double *out = a.partial + ((size_t)blockIdx.x * HQ_NL + lane) * HQ_NV;
#pragma unroll
        for (int v = 0; v < HQ_NV; v++) out[v] = 0.0;
#pragma unroll
        for (int v = 0; v < NB; v++) out[SL::slot(v)] = s[v];
    }
}

// ---------------------------------------------------------------------------
// Rate-program precompute (once per instance): Algorithm 3
// walked symbolically over the tile's varying units.
// ---------------------------------------------------------------------------
struct PairAcc3 {
    int n;
    uint32_t key[V3_MAXPAIRS / 4];   // unit | S << 6
    double val[V3_MAXPAIRS / 4];
};
constexpr int MAXP = V3_MAXPAIRS / 4;

__device__ __forceinline__ bool pair_add3(PairAcc3 &P, double *W0, int u, uint32_t S, double val) {
    if (S == 0u) {
        W0[u] += val;
        return true;
    }
    const uint32_t key = (uint32_t)u | (S << 6);
    for (int i = 0; i < P.n; i++)
        if (P.key[i] == key) {
            P.val[i] += val;
            return true;
        }
    if (P.n >= MAXP) return false;
    P.key[P.n] = key;
    P.val[P.n] = val;
    P.n++;
    return true;
}

__device__ bool tile_walk3(const P3Args &a, uint32_t t, double *W0, PairAcc3 &P) {
    const int NVU = 9 + a.nW;
    uint32_t Sst[HQ_MAXN + 2];
    Sst[0] = 0;
    for (int u = 0; u <= HQ_MAXN; u++) W0[u] = 0.0;
    P.n = 0;
    int v = 0;
    while (v < a.nnodes) {
        const int2 nd = __ldg(&a.node[v]);
        const int u = nd.x & 0xff;
        const int d = (nd.x >> 8) & 0xff;
        if (u >= NVU && !((t >> (u - NVU)) & 1u)) {   // tile unit, free in this tile: dead subtree
            v = nd.y;
            continue;
        }
        const uint32_t Spre = Sst[d - 1];
        const uint32_t own = u < NVU ? (1u << u) : 0u;
        if (!pair_add3(P, W0, u, Spre, __ldg(&a.lam_thr[v]))) return false;
        if (!a.full_lists) {
            const double e = __ldg(&a.lam_end[v]);
            if (e != 0.0 && !pair_add3(P, W0, a.N, Spre | own, e)) return false;
        }
        Sst[d] = Spre | own;
        v++;
    }
    return true;
}

__global__ void k_prog_count3(P3Args a, const uint32_t *__restrict__ order, uint32_t *__restrict__ size16,
                              int *__restrict__ err) {
    PairAcc3 P;
    double W0[HQ_MAXN + 1];
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.ntiles;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (!tile_walk3(a, order[i], W0, P)) {
            atomicExch(err, 2);
            size16[i] = V3_HDR16;
            continue;
        }
        int cnt[HQ_MAXN + 1][2];
        for (int u = 0; u <= HQ_MAXN; u++) cnt[u][0] = cnt[u][1] = 0;
        const uint32_t PR = 1u | (1u << 1) | (1u << 7) | (1u << 8);
        for (int k = 0; k < P.n; k++) cnt[P.key[k] & 63][((P.key[k] >> 6) & PR) ? 1 : 0]++;
        for (int u = 0; u <= HQ_MAXN; u++)
            if (cnt[u][0] > 255 || cnt[u][1] > 255) atomicExch(err, 3);
        size16[i] = V3_HDR16 + (uint32_t)P.n;
    }
}

__global__ void k_prog_write3(P3Args a, const uint32_t *__restrict__ order, const uint32_t *__restrict__ off16,
                              uint4 *__restrict__ prog) {
    PairAcc3 P;
    double W0[HQ_MAXN + 1];
    const int NVU = 9 + a.nW;
    const uint32_t PR = 1u | (1u << 1) | (1u << 7) | (1u << 8);
    uint32_t LW = 0;
    for (int u = 2; u <= 6; u++) LW |= 1u << u;
    for (int u = 9; u < NVU; u++) LW |= 1u << u;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.ntiles;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 *out = prog + off16[i];
        if (!tile_walk3(a, order[i], W0, P)) continue;
        // stable insertion sort by (unit, class): class 0 = lane-only, 1 = register-dependent
        auto rank = [&](uint32_t key) -> int { return (int)(key & 63) * 2 + ((((key >> 6) & PR) != 0u) ? 1 : 0); };
        for (int x = 1; x < P.n; x++) {
            const uint32_t kx = P.key[x];
            const double vx = P.val[x];
            const int rx = rank(kx);
            int y = x - 1;
            while (y >= 0 && rank(P.key[y]) > rx) {
                P.key[y + 1] = P.key[y];
                P.val[y + 1] = P.val[y];
                y--;
            }
            P.key[y + 1] = kx;
            P.val[y + 1] = vx;
        }
        uint32_t info[32];
        for (int q = 0; q < 32; q++) info[q] = 0u;
        for (int k = P.n - 1; k >= 0; k--) {   // start = index of the unit's first pair
            const int u = (int)(P.key[k] & 63);
            info[u] = (info[u] & 0xffffu) | ((uint32_t)k << 16);
        }
        for (int k = 0; k < P.n; k++) {
            const int u = (int)(P.key[k] & 63);
            const bool reg = ((P.key[k] >> 6) & PR) != 0u;
            info[u] += reg ? (1u << 8) : 1u;
        }
        for (int q = 0; q < 8; q++) out[q] = make_uint4(info[4 * q], info[4 * q + 1], info[4 * q + 2], info[4 * q + 3]);
        double *w0o = reinterpret_cast<double *>(out + 8);
        for (int u = 0; u < 32; u++) w0o[u] = u <= HQ_MAXN ? W0[u] : 0.0;
        for (int k = 0; k < P.n; k++) {
            const int u = (int)(P.key[k] & 63);
            const uint32_t S = P.key[k] >> 6;
            const bool pseudo = (u == a.N);
            uint32_t St = S & LW;
            if (!pseudo && ((LW >> u) & 1u)) St |= 1u << u;   // lane/warp unit: own busy condition
            uint32_t rm = 0xffffu;
            if ((S & PR) != 0u) {
                rm = 0u;
                for (int beta = 0; beta < 2; beta++)
                    for (int r = 0; r < R; r++) {
                        const int b0 = beta ^ (__popc(r) & 1);
                        bool ok = true;
                        if ((S & (1u << 1)) && !(r & 1)) ok = false;
                        if ((S & (1u << 7)) && !(r & 2)) ok = false;
                        if ((S & (1u << 8)) && !(r & 4)) ok = false;
                        if ((S & 1u) && !b0) ok = false;
                        if (!pseudo) {   // own busy condition of the parity / register units
                            if (u == 0 && !b0) ok = false;
                            if (u == 1 && !(r & 1)) ok = false;
                            if (u == 7 && !(r & 2)) ok = false;
                            if (u == 8 && !(r & 4)) ok = false;
                        }
                        if (ok) rm |= 1u << (r + 8 * beta);
                    }
            }
            const double c = P.val[k];
            out[V3_HDR16 + k] = make_uint4((uint32_t)__double_as_longlong(c),
                                           (uint32_t)((unsigned long long)__double_as_longlong(c) >> 32), St, rm);
        }
    }
}

}  // namespace hq3

// ---------------------------------------------------------------------------
namespace hq3_launch {

int choose_nw(int N) {
    int nw = N - 9 - 8;   // keep >= 256 tiles while the CTA is narrower than 16 warps
    if (nw < 0) nw = 0;
    if (nw > 4) nw = 4;
    if (nw > N - 9) nw = N - 9;
    return nw;
}

size_t sweep_smem(int nW, uint32_t maxrec16) {
    const size_t tstates = (size_t)1 << (8 + nW);
    return 2 * tstates * 8 + 2 * (size_t)maxrec16 * 16 + ((size_t)1 << nW) * V3_RING * V3_SLOT * 8;
}

cudaError_t prog_count(const P3Args &a, const uint32_t *order, uint32_t *size16, int *err, int grid, cudaStream_t s) {
    hq3::k_prog_count3<<<grid, 64, 0, s>>>(a, order, size16, err);
    return cudaGetLastError();
}
cudaError_t prog_write(const P3Args &a, const uint32_t *order, const uint32_t *off16, uint4 *prog, int grid,
                       cudaStream_t s) {
    hq3::k_prog_write3<<<grid, 64, 0, s>>>(a, order, off16, prog);
    return cudaGetLastError();
}

template <int MODE, bool FULL>
static cudaError_t launch(const S3Args &a, int grid, cudaStream_t s) {
    const size_t sm = sweep_smem(a.nW, a.maxrec16);
    cudaError_t e = cudaFuncSetAttribute(hq3::k_sweep3<MODE, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    hq3::k_sweep3<MODE, FULL><<<grid, 32 << a.nW, sm, s>>>(a);
    return cudaGetLastError();
}

cudaError_t sweep(const S3Args &a, int full, int mode, int grid, cudaStream_t s) {
    if (full) {
        if (mode == 0) return launch<0, true>(a, grid, s);
        if (mode == 1) return launch<1, true>(a, grid, s);
        return launch<2, true>(a, grid, s);
    }
    if (mode == 0) return launch<0, false>(a, grid, s);
    if (mode == 1) return launch<1, false>(a, grid, s);
    return launch<2, false>(a, grid, s);
}

}  // namespace hq3_launch
