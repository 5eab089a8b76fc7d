// hq_v3.h -- argument blocks and program format of the CTA-tiled sweep path
// (hq_v3.cu).  Product code only; nothing here is shared with oracle/.
//
// Tile geometry (compressed index j of a parity class):
//   bit 0            register bit 0   (internal unit 1)
//   bits 1..5        lane bits        (internal units 2..6)
//   bits 6..7        register bits 1-2 (internal units 7, 8)
//   bits 8..8+nW-1   warp bits        (internal units 9 .. 8+nW)
//   bits T.. (T=8+nW) tile index t    (internal units 9+nW .. N-1, "H" units)
// Internal unit 0 is the implied parity unit: b0 = c ^ parity(j).
// A CTA of 32 << nW threads owns one tile (2^T compressed states) at a time;
// thread (warp w, lane l) owns the 8 states r = 0..7 of its (w, l) slot.
// Rate programs are per warp tile (256 states, index t' = t << nW | w): only
// units 0..8 vary inside a program; units >= 9 are fixed by t'.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "hq_internal.h"

#define V3_R 8                 // states per thread
#define V3_HDR16 33            // program header: {info, M, W0} x 32 units, {mu_F, has}
#define V3_MAXPAIRS 2048

// rate program of a warp tile or of a CTA tile (16-byte records):
//   [0..31]  per unit u (u = N: blocked pseudo-unit): {info, M, W0 lo, W0 hi}
//            info = table << 31 | rtab << 30 | start << 8 | n_group (0: no data, W0 alone
//            applies); rtab: a register table follows the lane table (8 records: the summed
//            rate of the register-dependent pairs without lane / warp condition, per register
//            state r, for beta = 0 (records 0..3) and beta = 1 (records 4..7));
//            M = thread bits the unit's table is indexed by (lane bits 0..4, warp bits 5..8);
//            W0 = the tile-uniform rate of the unit
//   [32]     {mu_F lo, mu_F hi, has, 0}: mu_F = sum of nu over the busy tile units
//   data     per unit with data, at record 33 + start: a table of 2^|M| fp64 entries (if
//            info >> 31), the register table (if rtab), then n_group groups, each a header {rm | M_g << 16, 0, 0, 0} and a
//            table of 2^|M_g| entries; rm = admissible register states for beta = 0
//            (bits 0..7) and beta = 1 (bits 8..15).  A thread's entry is pext(thread bits, M).
// The programs of the warp tiles of a CTA tile (or its one CTA program) are contiguous.

// ---- device-resident solve (k_loop3): control block and exact phase sums
// Nonnegative per-layer sums in fixed point: HQ_XL 32-bit limbs in 64-bit words, unit
// 2^(xe - 32 HQ_XL); three rotating phase buffers.
#define HQ_XL 5
#define HQ_NX 8      // value slots: V2_P, V2_OM, V2_KA, V2_LAM, V2_DL1, residual num, den, -
enum { XV_RNUM = 5, XV_RDEN = 6 };
#define HQ_XG_WORDS (3 * HQ_NL * HQ_NX * HQ_XL)
struct Ctl3 {                    // written by CTA 0 when k_loop3 exits (host reads it once)
    int status;                  // SOLVE3_*
    int sweeps, halfsweeps, nres, phases, err;
    double updates, res, proxy;
    unsigned long long ns_sweep, ns_res;
};
enum { SOLVE3_RUNNING = 0, SOLVE3_CONVERGED = 1, SOLVE3_MAXITER = 2, SOLVE3_NUMERIC = 3, SOLVE3_NOTDECR = 4 };

struct S3Args {
    int N;
    int nW;                  // log2(warps per CTA)
    int c;                   // class updated (sweep) / evaluated (residual)
    uint32_t active;         // layers updated in this half-sweep
    uint64_t ntiles;
    uint64_t chunk;          // tiles per CTA (contiguous range of the visit order)
    double Lam;
    double nu[32];           // internal-order service rates
    const uint32_t *order;   // CTA-tile visit order (tile index t)
    const uint32_t *off16;   // [ntiles << nW]: program of warp w of visit index i at off16[i << nW | w]
                             // (CTA programs: the same offset for every warp of a tile)
    const uint4 *prog;
    uint32_t total16;
    uint32_t maxblk16;       // largest program block of a CTA tile (16-byte units)
    const uint32_t *range;   // [grid + 1]: CTA b processes visit indices [range[b], range[b+1])
    const double *Q;         // neighbour class (read)
    double *P;               // updated class (sweep) / evaluated class (residual)
    const double2 *omkap;    // scatter weights of class c
    const double *coef;      // v2 scalar block (V2S_* offsets)
    double *partial;         // MODE 2: [grid][HQ_NL][HQ_NV]; MODE 0/1: [HQ_NL][HQ_NV][grid]
    int full_lists;
    int warp_programs;       // 1: one rate program per warp tile (tables over lane bits only)
    int all_staged;          // 1: every tile's program block fits the staged capacity (maxblk16)
    unsigned long long *wtime;   // -DHQ_WARP_TIMING builds: busy cycles per (CTA, warp)
    // L2 policy of the tile-unit neighbour loads: units h < h_in (the tile bits of a group,
    // group order) evict-last; the others h_out_pol (0 evict-last, 1 evict-normal, 2 evict-first)
    int h_in;
    int h_out_pol;
    uint64_t pol[4];         // L2 policy encodings: evict-last, evict-normal, evict-first, half evict-last
    int in_pol;              // policy (index into pol) of the q blocks and the neighbours h < h_in
    // the three policies the sweep kernel uses, resolved by the host (plain parameters: the
    // cache-hinted loads take them from uniform registers without a per-load select)
    uint64_t pol_q;          // = pol[in_pol]: q blocks, tile-unit neighbours h < h_in
    uint64_t pol_hout;       // = pol[h_out_pol]: tile-unit neighbours h >= h_in
    uint64_t pol_ef;         // = pol[2]: streamed operands (programs, omega/kappa, stores)
    int pf_h;                // > 0: L2 prefetch of the tile-unit neighbour slices pf_h units ahead
    int pf_o;                // 1: L2 prefetch of the tile's scatter weights before the tile units
    int pf_min;              // prefetch only the tile units h >= pf_min
    // group progress bound (group order): CTA b's k-th tile is the
    // (b + k G)-th of the group-major sequence, group (b + k G) >> gs_bits.  A CTA adds 1 to
    // gs_ctr[g] once it is done with its tiles of group g (at once for groups it has no tile
    // in), and its thread 0 goes on with a tile of group g only when every CTA is done with
    // group g - gs_lag (gs_ctr[g - gs_lag] >= gs_target = launches x G: the counters are never
    // reset).  Only the visit timing changes, never a CTA's tiles or its summation order.
    // Needs every CTA resident (cooperative launch).
    unsigned long long *gs_ctr;   // [gs_ng] or nullptr (off)
    unsigned long long gs_target;
    int gs_bits, gs_lag;
    uint32_t gs_ng;
    // folded scalar step (MODE 0/1): every CTA first performs the scalar step of the previous
    // half-sweep (class prev_c, layers prev_active) from that launch's transposed partials
    // prev_partial and the block coef; CTA 0 stores the updated block in blk_out
    int fold;
    int prev_c;
    uint32_t prev_active;
    const double *prev_partial;
    double *blk_out;
    // device-resident solve (k_solve3): both classes, the control block, exact sums
    double *pw;                  // [2^N] both classes (class 0 first)
    const double2 *omkap_all;    // [2^N] scatter weights of both classes
    double *blk;                 // scalar block: the init block in, the final block out
    unsigned long long *xg;      // [HQ_XG_WORDS] exact phase sums (host zeroes them)
    Ctl3 *ctl;
    int xe;                      // fixed-point exponent of the exact sums
    double tol;
    int max_iter;
};

struct P3Args {   // program precompute (one program per warp tile or per CTA tile)
    int N;
    int nW;                  // log2(warps per CTA)
    int nwv;                 // warp bits varying inside a program: nW (CTA programs) or 0 (warp programs)
    int full_lists;
    uint64_t ntiles;
    double nu[32];           // internal-order service rates (mu_F in the header)
    int nnodes;
    const int2 *node;        // .x = unit | depth << 8, .y = skip
    const double *lam_thr;
    const double *lam_end;
    // pair cache (optional, ccap > 0): the count pass stores each program's sorted pairs
    // (<= ccap of them) and W0 so that the write pass does not walk the trie again
    int ccap;
    uint32_t *ckey;          // [ntiles][ccap]
    double *cval;            // [ntiles][ccap]
    uint16_t *crm;           // [ntiles][ccap]
    double *cW0;             // [ntiles][32]
    int *cn;                 // [ntiles]: number of pairs, -1 if not cached
};

namespace hq3_launch {
cudaError_t prog_count(const P3Args &a, const uint32_t *order, uint32_t *size16, int *err, int grid, cudaStream_t s);
cudaError_t prog_write(const P3Args &a, const uint32_t *order, const uint32_t *off16, uint4 *prog, int *err,
                       int grid, cudaStream_t s);
cudaError_t sweep(const S3Args &a, int full, int mode, int grid, cudaStream_t s);
cudaError_t policies(uint64_t *host4);   // the L2 policy encodings (S3Args::pol), cached per process
// device-resident solve (k_loop3): one cooperative launch runs every half-sweep, the
// convergence checks and the verification residual; grid = the CTA ranges (a.range)
cudaError_t loop(const S3Args &a, int full, int grid, cudaStream_t s);
int loop_occupancy(const S3Args &a, int full);   // co-resident CTAs per SM (0: does not fit)
size_t loop_smem(int nW, uint32_t maxblk16);
size_t sweep_smem(int nW, uint32_t maxblk16);
bool fits_smem(int nW, uint32_t maxblk16, bool dev_loop);   // the sweep (or device-loop) kernel's smem fits
uint32_t choose_cap(int nW, uint32_t maxblk16, bool dev_loop);
int choose_nw(int N);
int ctas_per_sm(int nW);   // CTAs per SM the sweep grid is sized for
}  // namespace hq3_launch
