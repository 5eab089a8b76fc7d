// hq_v2.h -- argument blocks and program format of the production sweep path
// (hq_v2.cu).  Product code only.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "hq_internal.h"

// Warp tile: 128 compressed states; internal units 0..7 vary inside a tile.
#define PROG_TB 7
#define PROG_TILE 128
#define PROG_NVARY 8
// Program record (16-byte units): [0..7] per-unit pair counts (u32 x 32:
// low 16 bits lane-only pairs, high 16 bits register-state pairs),
// [8..23] W0[32] (fp64; zero for the lane units 1..5, whose contributions are
// all pairs carrying the unit's own lane bit), then pairs
// {c: fp64, w: u32 = lane5 | rm(beta=0) << 8 | rm(beta=1) << 12 | unit << 16, pad}
// sorted by unit.  Unit index N is the "blocked" pseudo-unit (truncated
// lists): sum of lambda_j over atoms whose whole list is busy.
#define PROG_CNT16 8
#define PROG_HDR16 24
#define PROG_MAXPAIRS 1024

// per-layer values reduced by the sweep kernel
#define NV2 5
enum { V2_P = 0, V2_OM = 1, V2_KA = 2, V2_LAM = 3, V2_DL1 = 4 };
enum { V2_RNUM = 0, V2_RDEN = 1 };

struct PermArg {
    int p[32];   // internal unit -> ABI unit
};

struct P2Args {   // precompute kernels
    int N;
    int full_lists;
    uint64_t ntiles;
    double Lam;
    double nu[32];
    int nnodes;
    const int2 *node;        // .x = unit | depth << 8, .y = skip
    const double *lam_thr;
    const double *lam_end;
};

struct S2Args {   // sweep / residual kernel
    int N;
    int c;
    uint32_t active;         // layers updated in this half-sweep
    int full_lists;
    uint64_t ntiles;
    double Lam;
    double nu[32];
    const uint32_t *order;   // tile visit order (by popcount)
    const uint32_t *off16;   // program offsets (16-byte units), in visit order
    const uint4 *prog;
    uint32_t total16;        // program buffer size (16-byte units)
    uint32_t maxrec;         // largest program (16-byte units) = per-warp smem slot
    const double *Q;         // neighbour class
    double *P;               // updated class
    const double2 *omkap;    // scatter weights of the updated class
    const double *coef;      // device scalar block (see V2S_* offsets)
    double *partial;         // [grid][HQ_NL][HQ_NV]
};

// offsets inside the v2 device scalar block (doubles)
enum {
    V2S_LAM = 0,      // lambda(n)
    V2S_MU = 32,      // mu(n)
    V2S_ALPHA = 64,   // alpha(n) = mu*(n)/lambda(n-1) for the next half-sweep
    V2S_BETA = 96,    // beta(n)  = lambda(n)/mu(n+1)
    V2S_PN = 128,     // p(n), index n + 1 (so that n = -1 and n = N + 1 read 0): 34 slots
    V2S_OM = 176,     // sum_{l in C_n} p(l) omega(l)
    V2S_KA = 208,     // sum_{l in C_n} p(l) kappa(l)
    V2S_DL1 = 240,    // sum |dp| of the last update of layer n
    V2S_SUMP = 272,   // sum p of the last update of layer n
    V2S_RNUM = 304,   // residual numerator per layer
    V2S_RDEN = 336,   // residual denominator per layer
    V2S_MUSTAR = 368, // mu*(n) used by the last update of layer n
    V2S_MISC = 400,   // [0] err flag (as double), [1] residual, [2] proxy
    V2S_TOTAL = 416
};

namespace hq2_launch {
cudaError_t lambda_states(const P2Args &a, double *lamarr, int grid, cudaStream_t s);
cudaError_t omkap(const P2Args &a, const double *lamarr, double2 *omkap, int grid, cudaStream_t s);
cudaError_t prog_scan(const uint32_t *size16, uint32_t *off16, uint64_t n, void *tmp, size_t *tmp_bytes,
                      cudaStream_t s);
cudaError_t prog_max(const uint32_t *size16, uint32_t *out, uint64_t n, void *tmp, size_t *tmp_bytes, cudaStream_t s);
cudaError_t scalars(int N, int full_lists, double Lam, int mode, int c, uint32_t active, int ncta,
                    const double *partial, double *blk, cudaStream_t s, int transposed = 0,
                    double *blk_out = nullptr);   // blk_out: write the updated block there instead of in place
cudaError_t assemble(int N, const double *pw, const double *pn1, const int *perm, double *pi, int grid,
                     cudaStream_t s);
int sweep_grid(int nsm);
}  // namespace hq2_launch
