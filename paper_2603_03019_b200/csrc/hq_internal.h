// hq_internal.h -- data structures shared by the host orchestration (hq_api.cu)
// and the sm_100a kernels (hq_kernels.cu) of the B200 solver.  Product code:
// nothing here is shared with the CPU oracle (oracle/).
//
// Layout of the working set in HBM:
//   * parity-compressed natural order ("checkerboard"): states of even
//     popcount live in pw[0 .. 2^(N-1)), odd ones in pw[2^(N-1) .. 2^N).
//     Inside a class, state m sits at compressed index j = m >> 1; bit 0 of m
//     is implied by the class: b0 = c ^ parity(j).  All N single-bit-flip
//     neighbours of a class-c state are class-(1-c) states at j (unit 0) and
//     j ^ 2^(u-1) (unit u >= 1).  A red-black half-sweep therefore reads one
//     class and writes the other.
//   * pw holds the conditional probabilities p_n(B_m) (Proposition 1,
//     PAPER.md:216-224); pi is only assembled at the end.
//   * ab scratch: (a_m, b_m) of Eq. updateHeter for the class being updated.
#pragma once
#include <cstdint>

#define HQ_MAXN 31
#define HQ_NL 32               // layer slots (N + 1 <= 32)
#define HQ_BLOCK 256
#define HQ_NV 8                // per-layer reduction values per CTA

// Per-layer accumulator slots written by the sweep kernels.
enum {
    RV_SA = 0,    // sum a_m
    RV_SB = 1,    // sum b_m
    RV_SLA = 2,   // sum lambda_m a_m
    RV_SLB = 3,   // sum lambda_m b_m
    RV_SMA = 4,   // sum mu_m a_m
    RV_SMB = 5,   // sum mu_m b_m
};
enum {
    FV_DL1 = 0,   // sum |p_new - p_old|
    FV_DDEN = 1,  // sum (lambda_m + mu_m) |p_new - p_old|
    FV_SUMP = 2,  // sum p_new
};

struct NuArg {   // per-unit rates by value (N <= 31)
    double v[32];
};

struct DevTrie {
    int nnodes;
    const int2 *node;        // .x = unit of the node, .y = preorder index after its subtree
    const double *lam_thr;   // Lambda_v = sum of lambda_j over atoms whose list passes through v
    const double *lam_end;   // sum of lambda_j over atoms whose list ends at v (truncated lists)
};

struct KArgs {
    int N;
    int c;                   // class being updated / processed
    uint32_t active;         // bit n set: layer n is updated in this half-sweep
    int full_lists;
    uint64_t nstates_c;      // 2^(N-1): states per class
    uint64_t ntiles;
    double Lam;
    double nu[32];
    DevTrie trie;
    const double *Q;         // neighbour class (read)
    double *P;               // updated class (read old / write new)
    double2 *ab;             // scratch (a, b) per state of the updated class
    const double *lam_n;     // [HQ_NL] lambda(n) (latest)
    const double *mu_n;      // [HQ_NL] mu(n) (latest)
    const double *mustar;    // [HQ_NL] mu*(n) of this half-sweep
    const double *pn;        // [HQ_NL] layer masses p(n) (residual / assembly)
    double *partial;         // [grid][HQ_NL][HQ_NV]
    const double2 *omkap;    // v2 init: scatter weights of class c
    const double *lamarr;    // v2 init (truncated lists): lambda_m of class c, or NULL
};
