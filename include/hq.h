/*
 * hq.h -- C-ABI of the B200-native steady-state solver for the spatial
 * hypercube queueing model with heterogeneous service rates
 * (arXiv 2603.03019; PAPER.md = the paper's text).
 *
 * The library (libhq.so, built from paper_2603_03019_b200/csrc) runs every
 * step of the solve in hand-written sm_100a CUDA kernels.  There is no CPU
 * fallback: on a machine without a usable CUDA device every compute call
 * returns HQ_E_CUDA.
 *
 * Model.  N units, J demand atoms.  State m in [0, 2^N):
 * bit u of m is 1 iff unit u (0-based) is busy, i.e. the paper's index
 * y(B_m) with paper unit i = u + 1.  An arrival at atom j
 * (rate lambda[j] = lambda * f_j) is served by the first free unit of the
 * atom's preference list (Eq. tran_rates); if every unit of
 * the list is busy the call is lost (C = 0).  A busy
 * unit u completes service at rate mu[u] (the paper's nu_i).
 *
 * Thread safety: calls on different handles may run concurrently; calls on
 * one handle must be serialised by the caller.
 */
#ifndef HQ_H
#define HQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hq_problem *hq_handle;

typedef enum {
    HQ_OK = 0,
    HQ_NOT_CONVERGED = 1, /* warning: max_iter reached; outputs hold the last iterate */
    HQ_E_INVAL = -1,      /* invalid argument; see hq_error_string                     */
    HQ_E_NOMEM = -2,      /* device memory for the working set could not be allocated  */
    HQ_E_CUDA = -3,       /* CUDA runtime / launch error (or no device)                */
    HQ_E_NUMERIC = -4,    /* NaN/Inf or a non-positive normaliser in the iteration     */
    HQ_E_ORDER = -5       /* hq_measures before a successful hq_solve on this handle  */
} hq_status;

/*
 * hq_create -- validate an instance and build its device-side tables
 * (preference trie for on-the-fly upward rates, service rates).
 *
 *   N       number of units, 1 <= N <= 31 (2^31 states, 17.2 GB fp64 pi).
 *   J       number of demand atoms, J >= 1.
 *   lambda  [J] host, per-atom arrival rates lambda_j = lambda * f_j
 *           (PAPER.md:76, 96-97); each finite and >= 0, sum > 0.
 *   mu      [N] host, per-unit service rates (the paper's nu_i,
 *           PAPER.md:99); each finite and > 0.
 *   pref    [J][N] host, row-major int32: pref[j*N + h] is the 0-based id of
 *           the (h+1)-th preferred unit of atom j (the paper's zeta_j(h+1),
 *           PAPER.md:93).  A row may end early with -1 padding (truncated
 *           list: the call is lost when all listed units are busy).  Entries
 *           must be in [0, N), distinct within a row, no entry after a -1,
 *           rows non-empty.  Every unit must appear in the list of some atom
 *           with lambda_j > 0 (otherwise the chain is reducible and the
 *           stationary distribution is not unique).
 *   out     receives the handle.
 *
 * Ownership: the input arrays are copied; the caller may free them on
 * return.  The handle owns all device tables and scratch (allocated on the
 * current device at the first hq_solve), released by hq_destroy.
 * Errors: HQ_E_INVAL (message via hq_error_string(NULL)), HQ_E_CUDA.
 */
hq_status hq_create(int N, int J, const double *lambda, const double *mu, const int32_t *pref, hq_handle *out);

/*
 * hq_solve -- the layer-ordered conditional-probability iteration
 * (Algorithm 1, Eqs. updateHeter / lambdaHeter / muHeter,
 * PAPER.md:313-320) to a relative balance residual <= tol, then the
 * assembly P{B_m} = p(w(B_m)) p_{w(B_m)}(B_m) (Proposition 1, PAPER.md:224,
 * Eq. bnd_stationary).
 *
 *   tol       target of the relative L1 global-balance residual
 *             r(pi) = sum_m |pi(m)(lambda_m + mu_m) - inflow(m)| /
 *                     sum_m pi(m)(lambda_m + mu_m)        (Eq. balance_eq_heter,
 *             PAPER.md:161; reading R3).  tol <= 0 runs exactly
 *             max_iter sweeps.
 *   max_iter  maximum number of sweeps (each sweep updates layers 1..N-1
 *             once, i.e. 2^N - 2 states).
 *   pi        [2^N] DEVICE fp64, caller-owned (e.g. a torch.float64 CUDA
 *             tensor); on return pi[m] = P{B_m} at natural index m.
 *   cuda_stream  cudaStream_t to run on (NULL = legacy default stream).
 *   iters_out    host: sweeps performed.
 *   residual_out host: the true r(pi) of the returned pi (not a proxy).
 *
 * Execution: N >= 9 runs the CTA-tiled sweep kernel; for N < 21
 * the whole loop -- every half-sweep, the convergence checks and the verification
 * residual -- is ONE cooperative launch (device-resident; the host synchronises
 * once), for N >= 21 one launch per half-sweep with host-scheduled checks (the
 * faster path there); HQ_LOOP=device|host in the environment at hq_create forces
 * either.  An instance whose per-tile rate programs exceed their format (more than
 * 2048 distinct (unit, condition) pairs in a tile, e.g. thousands of unstructured
 * lists) falls back to the general two-pass path (per-thread trie walk; slower).
 *
 * Device memory (allocated at the first hq_solve, from the CUDA memory pool):
 * 8 B/state for the conditional probabilities p_n + 16 B/state of scatter weights
 * (+ 8 B/state of lambda_m for truncated lists) + the rate programs (hq_stats [12];
 * about 4 B/state at the BASELINE configs) + small tables, i.e. about 28-36 B x 2^N
 * (75-77 GB at N = 31), plus the caller's pi (8 B x 2^N).  N is at most 31
 * (HQ_MAXN); HQ_E_NOMEM if the working set does not fit the free device memory.
 *
 * The call synchronises cuda_stream before returning.
 * Returns HQ_OK, HQ_NOT_CONVERGED (pi, iters, residual hold the last
 * iterate), HQ_E_INVAL, HQ_E_NOMEM, HQ_E_CUDA or HQ_E_NUMERIC (a non-positive or
 * non-finite layer normaliser, a non-finite sum, or a convergence proxy that grew by
 * more than 1.5x at four consecutive checks: the iteration diverges -- Assumption 1,
 * PAPER.md:359-367, is not guaranteed for every instance).
 */
hq_status hq_solve(hq_handle h, double tol, int max_iter, double *pi, void *cuda_stream, int *iters_out,
                   double *residual_out);

/*
 * hq_measures -- performance measures of a stationary distribution pi
 * (device, natural index, normally the output of hq_solve on this handle).
 *
 *   workload  [N] DEVICE fp64: rho_i = P(unit i busy) = sum_{m: bit i} pi(m)
 *             ("Unit Utilization").
 *   dispatch  [J*N] DEVICE fp64, row-major [j][i]: the fraction of served
 *             calls that come from atom j and are served by unit i,
 *             rho_ij = f_j sum_{m in S_ij} pi(m) / (1 - loss), S_ij = states in
 *             which i is atom j's first free unit (PAPER.md:787-789,
 *             1759-1761); sum_ij rho_ij = 1.  Zero for units not in the list.
 *   loss      host scalar: fraction of arrivals lost,
 *             sum_j f_j P(every unit of list j busy) (= P{all busy} for full
 *             lists, the paper's Pi).
 *   cuda_stream  as in hq_solve; the call synchronises it before returning.
 * Returns HQ_OK, HQ_E_ORDER (no successful hq_solve yet), HQ_E_INVAL,
 * HQ_E_NOMEM, HQ_E_CUDA.  The size of pi cannot be checked: it is the
 * caller's contract.
 */
hq_status hq_measures(hq_handle h, const double *pi, double *workload, double *dispatch, double *loss,
                      void *cuda_stream);

/*
 * hq_response_times -- response-time measures (SURVEY.md
 * §8(f) row f3) of the zero-capacity system from the dispatch fractions of
 * hq_measures:
 *   MRT   = sum_ij rho_ij tau_ij            MRT_j = sum_i rho_ij tau_ij / sum_i rho_ij
 *   F(T)  = sum_j f_j P{E(j, T)} / (1 - Pi) F_j(T) = P{E(j, T)} / (1 - Pi)
 * where E(j, T) = union_i {m in S_ij : tau_ij < T} (strict), so
 * F(T) = sum_{ij: tau_ij < T} rho_ij and F_j(T) = sum_{i: tau_ij < T} rho_ij / f_j.
 *
 *   dispatch  [J*N] DEVICE: rho_ij as written by hq_measures on this handle.
 *   tau       [J*N] host, row-major [j][i]: response time of unit i to atom j
 *             (finite, >= 0; units of the caller's choice).
 *   T_bar     threshold T.
 *   mrt, frac_within  host scalars: MRT and F(T_bar).
 *   mrt_j, frac_within_j  [J] DEVICE or NULL: MRT_j and F_j(T_bar) (0 for an atom
 *             with f_j = 0).
 * Errors: HQ_E_INVAL (NULL, NaN, negative tau, or a waiting room is set: the paper
 * defines these measures for C = 0), HQ_E_NOMEM, HQ_E_CUDA.
 */
hq_status hq_response_times(hq_handle h, const double *dispatch, const double *tau, double T_bar, double *mrt,
                            double *frac_within, double *mrt_j, double *frac_within_j, void *cuda_stream);

/*
 * hq_set_buffer -- give calls that find every unit busy a waiting room
 * (SURVEY.md §8(f) row f1).
 *
 *   C  0 (default): loss system, the model above.
 *      C > 0: finite buffer of C waiting calls (Proposition "Reformulation,
 *      Finite Buffer"): a call arriving when all N units
 *      are busy waits if fewer than C calls wait, otherwise it is lost;
 *      waiting calls are served first-come-first-served.
 *      HQ_BUFFER_UNLIMITED: unlimited waiting room (Remark);
 *      hq_solve then needs Lambda < sum of the service rates.
 *
 * Needs full preference lists (every row of pref ranks all N units): a call
 * queues exactly when all N units are busy.  The
 * conditional probabilities p_n(B_m) are those of the loss system (the
 * proposition's update equations are unchanged); hq_solve then returns the
 * hypercube part P{B_m} = p(w(B_m)) p_w(B_m)(B_m) with the layer masses p(n)
 * of the extended birth-death chain, lambda(n) = Lambda and mu(n) = sum nu for
 * n > N, i.e. the loss-system pi scaled by 1 / (1 + P{all busy} sum_c r^c),
 * r = Lambda / sum nu.  residual_out stays the residual of the hypercube block,
 * an upper bound of the residual of the whole chain (the tail states satisfy
 * their balance equations in closed form; R15).  hq_measures
 * reports: workload includes the waiting states (all units busy); loss =
 * P~{C} (0 when unlimited); dispatch counts a queued call for the unit that
 * completes service first (unit i with probability nu_i / sum nu, DESIGN.md
 * R14), so sum_ij rho_ij = 1 and nu_i rho_i = Lambda (1 - loss) sum_j rho_ij.
 *
 * Takes effect at the next hq_solve (it invalidates the last one).
 * Errors: HQ_E_INVAL (C < HQ_BUFFER_UNLIMITED, or C != 0 with truncated lists).
 */
#define HQ_BUFFER_UNLIMITED (-1)
hq_status hq_set_buffer(hq_handle h, int C);

/*
 * hq_queue_tail -- after hq_solve with a waiting room: tail[c-1] = P~{c}, the
 * probability that c calls wait (P~{c} = p(N + c)), for
 * c = 1..len (host array, caller-owned; len <= C for a finite buffer; any len
 * when unlimited).  mass (host, may be NULL) receives sum_{c>=1} P~{c}.  With
 * C = 0 the tail is zero.  Errors: HQ_E_INVAL, HQ_E_ORDER (no solve yet).
 */
hq_status hq_queue_tail(hq_handle h, double *tail, int len, double *mass);

/*
 * hq_batch_solve -- many small instances in one call:
 * the paper's usage pattern of load sweeps (9 values per N)
 * and configuration screening (thousands of N = 9-11 solves).
 * One CTA per instance with its whole state space in shared memory; Algorithm 1
 * literally: layers 1..N-1 in order within a sweep, Eq.
 * updateHeter with the inner normalisation limit (R1), Eqs.
 * lambdaHeter / muHeter after each layer, Eq. bnd_stationary for p(n); the
 * relative balance residual r(pi) (R3) every 4 sweeps; stop at r <= tol.
 *
 *   B, N, J   instances, units (1 <= N <= 12), atoms (pad with lambda = 0 atoms
 *             to a common J).
 *   lambda    [B][J] host, mu [B][N] host, pref [B][J][N] host (int32, -1
 *             padded rows allowed), each instance validated as in hq_create.
 *   tol, max_iter  as in hq_solve (max_iter >= 1).
 *   pi        [B][2^N] DEVICE fp64, caller-owned: pi[b*2^N + m] = P{B_m}.
 *   cuda_stream    stream to run on; the call synchronises it.
 *   iters_out, residual_out, status_out  [B] host (may be NULL): sweeps, true
 *             r(pi) of the returned pi, HQ_OK / HQ_NOT_CONVERGED / HQ_E_NUMERIC.
 *   workload  [B][N] DEVICE or NULL, dispatch [B][J][N] DEVICE or NULL,
 *   loss_out  [B] host or NULL: the measures of hq_measures per instance, computed
 *             on chip from the instance's pi (superset sums, fixed order).
 * Returns the worst per-instance status, or HQ_E_INVAL / HQ_E_CUDA (message via
 * hq_batch_error_string).  Scratch (B * 2^N * N fp64 dispatch rates) is
 * allocated and freed inside the call.
 */
hq_status hq_batch_solve(int B, int N, int J, const double *lambda, const double *mu, const int32_t *pref,
                         double tol, int max_iter, double *pi, void *cuda_stream, int *iters_out,
                         double *residual_out, int *status_out, double *workload, double *dispatch,
                         double *loss_out);
const char *hq_batch_error_string(void);

/* Release every device and host resource of h (NULL is a no-op). */
void hq_destroy(hq_handle h);

/* Last error text for h; h == NULL returns the last hq_create error. */
const char *hq_error_string(hq_handle h);

/*
 * Introspection for tests and the benchmark (not part of the paper's
 * problem statement).  hq_stats fills a host array of HQ_STATS_LEN doubles
 * describing the last hq_solve:
 *   [0] sweeps, [1] half-sweeps, [2] state updates (sum over updated layers
 *   of C(N,n)), [3] kernel launches, [4] true-residual evaluations,
 *   [5] trie nodes, [6] sum(pi) - 1, [7] solve time in ms (CUDA events),
 *   [8] time in the sweep kernels in ms (CUDA events), [9] sweep-kernel
 *   launches, [10] residual-kernel time in ms, [11] one-off per-instance
 *   precompute time in ms (rate programs, scatter weights), [12] bytes of
 *   rate programs, [13] code path (1: N < 9 two-pass or the fallback, 3: CTA-tiled),
 *   [14] largest rate-program block of a CTA tile (16-byte records),
 *   [15] warp bits varying inside a rate program (0: one program per warp tile,
 *        the default; nW: one program per CTA tile, HQ_PROG=cta),
 *   [16] device-resident solve: time of its one k_solve3 launch in ms (CUDA events),
 *   [17] 1 if the solve ran device-resident (one launch for every half-sweep, check and
 *        residual; [8] and [10] then split [16] by the phases' timestamps), 0 if host-looped,
 *   [18] tile visit order of the CTA-tiled path: -1 popcount order, b >= 0 chunked
 *        order with chunks of 2^b tiles (N >= 27),
 *   [19] group progress bound of the group order: a CTA starts a tile of group g only
 *        when every CTA is done with group g - [19] (0: unbounded).
 */
#define HQ_STATS_LEN 20
hq_status hq_stats(hq_handle h, double *out);

/* Copy an internal device array to host memory (tests and debugging only):
 * which = 0 scalar block, 1 conditional probabilities, 2 scatter weights,
 * 3 rate programs, 4 program offsets, 5 tile order, 6 internal->ABI unit map.
 * Returns HQ_E_ORDER if the array does not exist yet. */
hq_status hq_debug_copy(hq_handle h, int which, void *host, size_t bytes);

/* Library build string (compiler, arch, git-independent version tag). */
const char *hq_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HQ_H */
