/*
 * hq_oracle.c -- plain, slow, obviously-correct CPU oracle for the spatial
 * hypercube queueing model with heterogeneous service rates
 * (arXiv 2603.03019, PAPER.md = /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2603_03019_b200/csrc); neither side includes the other.
 *
 * Conventions: unit u (0-based) <-> bit u of the
 * natural state index m = sum_u b_u 2^u (the paper's y(B_m), PAPER.md:536-539,
 * with paper unit i = u+1).  pref[j*N + h] is the h-th preferred unit of atom
 * j (the paper's zeta_j(h+1)), -1 padded for truncated lists
 * (SURVEY.md §8(c) C2).  lam[j] = lambda * f_j.
 *
 * All arithmetic is IEEE fp64; sums over states are accumulated serially in
 * ascending state order (no blocking, no reordering), so the result does not
 * depend on the thread count.  OpenMP is used only for loops whose iterations
 * write disjoint outputs.
 *
 * Functions and the passages they follow:
 *   oracle_dispatch_rates   Algorithm 3 read with
 *                           for state m and atom j the
 *                           units zeta_j(1..) up to and EXCLUDING the first
 *                           free unit receive lambda_j as the upward rate
 *                           lambda_{m\i -> m}; equals Eq. tran_rates
 *                            with the product read over
 *                           r < eta_j(i).
 *   oracle_out_rates        Eq. tran_rates seen from the source state l: each
 *                           atom sends lambda_j to its first free unit
 *                           ("the available unit with the highest
 *                           preference"); lost if none (C = 0,
 *                           PAPER.md:78, 165).
 *   oracle_solve            Algorithm 1 with Eqs.
 *                           updateHeter / lambdaHeter / muHeter
 *                           (PAPER.md:313-320), Eq. bnd_stationary
 *                            and Proposition 1
 *                           (PAPER.md:216-224); readings C1, C2, C3, C8, C9.
 *   oracle_residual         relative L1 global-balance residual of Eq.
 *                           balance_eq_heter, reading C3.
 *   oracle_measures         utilisation rho_i, dispatch
 *                           fractions rho_ij over S_ij and Pi
 *                           (PAPER.md:787-789, 1759-1761), readings C12, C13.
 *   oracle_residual_stream  the same residual with O(2^N / 2^B) scratch and the
 *                           rates of Eq. tran_rates taken through a prefix tree of
 *                           the lists (full-size checks, N up to 31).
 *   oracle_state_balance    the same balance equation at caller-chosen states
 *                           (sampled parity checks at sizes where a full
 *                           oracle run is infeasible).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_NOT_CONVERGED 1
#define ORACLE_E_INVAL (-1)
#define ORACLE_E_NOMEM (-2)

typedef struct {
    int N, J;
    const double *lam;   /* [J] */
    const double *mu;    /* [N] */
    const int32_t *pref; /* [J*N] */
} inst_t;

static int popcount64(uint64_t x) { return __builtin_popcountll(x); }

/* ---------------------------------------------------------------------- */
/* Rates                                                                   */
/* ---------------------------------------------------------------------- */

/* Algorithm 3 for one state m: W[i] = upward rate
 * lambda_{m\i -> m} for every busy unit i of m (0 for free units).
 * For atom j, zeta'_j = the units of zeta_j up to, excluding, the first unit
 * absent from U(B_m) (reading C6); each gets lambda_j. */
static void dispatch_rates(const inst_t *I, uint64_t m, double *W) {
    for (int i = 0; i < I->N; i++) W[i] = 0.0;
    for (int j = 0; j < I->J; j++) {
        for (int h = 0; h < I->N; h++) {
            int u = I->pref[(size_t)j * I->N + h];
            if (u < 0) break;                 /* truncated list exhausted */
            if (!((m >> u) & 1)) break;       /* first free unit: stop, exclusive */
            W[u] += I->lam[j];
        }
    }
}

/* Eq. tran_rates from the source side: out[i] = lambda_{l -> l+i} for every
 * free unit i of l; lost[0] = sum of lambda_j over atoms with no free unit
 * in their list (calls lost, C = 0). */
static void out_rates(const inst_t *I, uint64_t l, double *out, double *lost) {
    for (int i = 0; i < I->N; i++) out[i] = 0.0;
    double ls = 0.0;
    for (int j = 0; j < I->J; j++) {
        int found = -1;
        for (int h = 0; h < I->N; h++) {
            int u = I->pref[(size_t)j * I->N + h];
            if (u < 0) break;
            if (!((l >> u) & 1)) { found = u; break; }
        }
        if (found >= 0) out[found] += I->lam[j];
        else ls += I->lam[j];
    }
    *lost = ls;
}

/* lambda_m = total upward rate out of m (Table 1) and
 * mu_m = sum of nu_i over busy units. */
static double lambda_m(const inst_t *I, uint64_t m) {
    double tot = 0.0;
    for (int j = 0; j < I->J; j++) {
        for (int h = 0; h < I->N; h++) {
            int u = I->pref[(size_t)j * I->N + h];
            if (u < 0) break;
            if (!((m >> u) & 1)) { tot += I->lam[j]; break; }
        }
    }
    return tot;
}

static double mu_m(const inst_t *I, uint64_t m) {
    double s = 0.0;
    for (int i = 0; i < I->N; i++)
        if ((m >> i) & 1) s += I->mu[i];
    return s;
}

int oracle_dispatch_rates(int N, int J, const double *lam, const int32_t *pref, uint64_t m, double *W) {
    inst_t I = {N, J, lam, NULL, pref};
    dispatch_rates(&I, m, W);
    return ORACLE_OK;
}

int oracle_out_rates(int N, int J, const double *lam, const int32_t *pref, uint64_t l, double *out, double *lost) {
    inst_t I = {N, J, lam, NULL, pref};
    out_rates(&I, l, out, lost);
    return ORACLE_OK;
}

/* ---------------------------------------------------------------------- */
/* Layer enumeration                                                       */
/* ---------------------------------------------------------------------- */

static double binom(int n, int k) {
    if (k < 0 || k > n) return 0.0;
    double r = 1.0;
    for (int i = 1; i <= k; i++) r = r * (double)(n - k + i) / (double)i;
    return floor(r + 0.5);
}

/* states of layer C_n in ascending order (Gosper's hack). */
static uint64_t *layer_states(int N, int n, uint64_t *count) {
    uint64_t c = (uint64_t)binom(N, n);
    uint64_t *s = (uint64_t *)malloc(sizeof(uint64_t) * (c ? c : 1));
    if (!s) return NULL;
    if (n == 0) { s[0] = 0; *count = 1; return s; }
    uint64_t x = (1ULL << n) - 1, lim = 1ULL << N;
    uint64_t k = 0;
    while (x < lim) {
        s[k++] = x;
        uint64_t cc = x & (~x + 1), r = x + cc;
        x = (((r ^ x) >> 2) / cc) | r;
    }
    *count = k;
    return s;
}

/* ---------------------------------------------------------------------- */
/* Per-state coefficients, optionally cached                               */
/* ---------------------------------------------------------------------- */

typedef struct {
    const inst_t *I;
    double *Wtab;    /* [2^N * N] cached Algorithm 3 output, or NULL */
    double *lamtab;  /* [2^N] lambda_m, or NULL */
    double *mutab;   /* [2^N] mu_m, or NULL */
} rates_t;

static void state_W(const rates_t *R, uint64_t m, double *W) {
    if (R->Wtab) memcpy(W, R->Wtab + m * (uint64_t)R->I->N, sizeof(double) * R->I->N);
    else dispatch_rates(R->I, m, W);
}

static double state_lambda(const rates_t *R, uint64_t m) {
    return R->lamtab ? R->lamtab[m] : lambda_m(R->I, m);
}

static double state_mu(const rates_t *R, uint64_t m) {
    return R->mutab ? R->mutab[m] : mu_m(R->I, m);
}

/* ---------------------------------------------------------------------- */
/* Algorithm 1                                                             */
/* ---------------------------------------------------------------------- */

/* Eq. bnd_stationary given lam_n[0..N], mu_n[0..N]. */
static void birth_death(int N, const double *lam_n, const double *mu_n, double *pn) {
    double prod = 1.0, tot = 1.0;
    double *g = (double *)malloc(sizeof(double) * (N + 1));
    g[0] = 1.0;
    for (int n = 1; n <= N; n++) {
        prod *= lam_n[n - 1] / mu_n[n];
        g[n] = prod;
        tot += prod;
    }
    for (int n = 0; n <= N; n++) pn[n] = g[n] / tot;
    free(g);
}

/* Relative L1 global-balance residual of Eq. balance_eq_heter (reading C3):
 * r = sum_m |pi(m)(lambda_m+mu_m) - up-inflow - down-inflow| / sum_m pi(m)(lambda_m+mu_m). */
static double residual(const rates_t *R, const double *pi) {
    const inst_t *I = R->I;
    int N = I->N;
    uint64_t S = 1ULL << N;
    double *rm = (double *)malloc(sizeof(double) * S);
    double *om = (double *)malloc(sizeof(double) * S);
    if (!rm || !om) { free(rm); free(om); return NAN; }
#pragma omp parallel
    {
        double W[64];
#pragma omp for schedule(static)
        for (int64_t mm = 0; mm < (int64_t)S; mm++) {
            uint64_t m = (uint64_t)mm;
            state_W(R, m, W);
            double lm = state_lambda(R, m);
            double out = pi[m] * (lm + state_mu(R, m));
            double in = 0.0;
            for (int i = 0; i < N; i++) {
                uint64_t l = m ^ (1ULL << i);
                if ((m >> i) & 1) in += pi[l] * W[i];   /* upward transition into m   */
                else in += pi[l] * I->mu[i];             /* downward transition into m */
            }
            rm[m] = fabs(out - in);
            om[m] = out;
        }
    }
    double num = 0.0, den = 0.0;
    for (uint64_t m = 0; m < S; m++) { num += rm[m]; den += om[m]; }
    free(rm); free(om);
    return num / den;
}

/*
 * Algorithm 1.
 *   step 2: p_n^1(B_m) = 1/C(N,n); lambda^1(n), mu^1(n) by Eqs. lambdaHeter /
 *           muHeter on the uniform p (reading C8).
 *   steps 3-15: sweep k: for n = 1..N-1 ascending:
 *           a_m, b_m from Eq. updateHeter: p_n^{k,r} = mu^{k,r-1}(n) a_m + b_m,
 *             a_m = sum_{l in C_{n-1}} p_{n-1}^k(l) lambda_lm / (lambda^k(n-1) (lambda_m+mu_m))
 *             b_m = lambda^{k-1}(n)/mu^{k-1}(n+1) * sum_{l in C_{n+1}^m} p_{n+1}^{k-1}(l) mu_lm / (lambda_m+mu_m)
 *           inner r-loop: mu^{k,r}(n) = sum_m mu_m p_n^{k,r}(m),
 *             started at mu^{k,0}(n) = mu^{k-1}(n); since p^{k,r} is affine in
 *             mu^{k,r-1} the loop is run on the scalar (reading C1) until
 *             max_m |p^{k,r}-p^{k,r-1}| = |dmu| max_m a_m <= delta, delta = 0
 *             (i.e. until it stops changing), capped at 100000 steps;
 *           then p_n is renormalised to sum 1 (reading C2; a rounding-level
 *             no-op for full preference lists, Lemma 1);
 *           lambda^k(n) by Eq. lambdaHeter, mu^k(n) by Eq. muHeter
 *             (PAPER.md:348).
 *   stopping: after every sweep pi is assembled by Proposition 1 and
 *           Eq. bnd_stationary and the sweep loop stops when the residual
 *           r(pi) <= tol (reading C3) or after max_iter sweeps.
 * pi_out [2^N] receives P{B_m} (natural index).  trace (optional, [max_iter])
 * receives r(pi) after each sweep.
 */
int oracle_solve(int N, int J, const double *lam, const double *mu, const int32_t *pref,
                 double tol, int max_iter, int use_table, double *pi_out, int *iters_out,
                 double *residual_out, double *trace, double *layer_lam_out, double *layer_mu_out) {
    if (N < 1 || N > 31 || J < 1) return ORACLE_E_INVAL;
    inst_t I = {N, J, lam, mu, pref};
    uint64_t S = 1ULL << N;
    rates_t R = {&I, NULL, NULL, NULL};
    /* per-state lambda_m and mu_m are cached (same arithmetic, computed once) */
    R.lamtab = (double *)malloc(sizeof(double) * S);
    R.mutab = (double *)malloc(sizeof(double) * S);
    if (!R.lamtab || !R.mutab) { free(R.lamtab); free(R.mutab); return ORACLE_E_NOMEM; }
    if (use_table) {
        R.Wtab = (double *)malloc(sizeof(double) * S * (uint64_t)N);
        if (!R.Wtab) { free(R.lamtab); free(R.mutab); return ORACLE_E_NOMEM; }
    }
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < (int64_t)S; m++) {
        if (R.Wtab) dispatch_rates(&I, (uint64_t)m, R.Wtab + (uint64_t)m * N);
        R.lamtab[m] = lambda_m(&I, (uint64_t)m);
        R.mutab[m] = mu_m(&I, (uint64_t)m);
    }

    double *p = (double *)malloc(sizeof(double) * S);   /* p_n(B_m) at natural index m */
    double *a = (double *)malloc(sizeof(double) * S);
    double *b = (double *)malloc(sizeof(double) * S);
    uint64_t **lay = (uint64_t **)calloc(N + 1, sizeof(uint64_t *));
    uint64_t *cnt = (uint64_t *)calloc(N + 1, sizeof(uint64_t));
    double *lam_n = (double *)calloc(N + 1, sizeof(double));
    double *mu_n = (double *)calloc(N + 1, sizeof(double));
    double *pn = (double *)calloc(N + 1, sizeof(double));
    if (!p || !a || !b || !lay || !cnt || !lam_n || !mu_n || !pn) return ORACLE_E_NOMEM;
    for (int n = 0; n <= N; n++) {
        lay[n] = layer_states(N, n, &cnt[n]);
        if (!lay[n]) return ORACLE_E_NOMEM;
    }

    /* step 2: uniform conditional probabilities and the initial layer rates */
    for (int n = 0; n <= N; n++) {
        double v = 1.0 / (double)cnt[n];
        for (uint64_t t = 0; t < cnt[n]; t++) p[lay[n][t]] = v;
    }
    for (int n = 0; n <= N; n++) {
        double sl = 0.0, sm = 0.0;
        for (uint64_t t = 0; t < cnt[n]; t++) {
            uint64_t m = lay[n][t];
            sl += p[m] * state_lambda(&R, m);
            sm += p[m] * state_mu(&R, m);
        }
        lam_n[n] = sl;   /* Eq. lambdaHeter; lambda(N) = 0 for C = 0 full lists */
        mu_n[n] = sm;    /* Eq. muHeter; mu(0) = 0 */
    }

    int k = 0, status = ORACLE_NOT_CONVERGED;
    double res = NAN;
    while (k < max_iter) {
        k++;
        for (int n = 1; n <= N - 1; n++) {
            const uint64_t *L = lay[n];
            const uint64_t c = cnt[n];
            const double lam_prev = lam_n[n - 1];        /* lambda^k(n-1), reading C9 */
            const double ratio = lam_n[n] / mu_n[n + 1];  /* lambda^{k-1}(n)/mu^{k-1}(n+1) */
#pragma omp parallel
            {
                double W[64];
#pragma omp for schedule(static)
                for (int64_t t = 0; t < (int64_t)c; t++) {
                    uint64_t m = L[t];
                    state_W(&R, m, W);
                    double up_in = 0.0, down_in = 0.0;
                    for (int i = 0; i < N; i++) {
                        uint64_t l = m ^ (1ULL << i);
                        if ((m >> i) & 1) up_in += p[l] * W[i];   /* l in C_{n-1}, lambda_lm = W[i] */
                        else down_in += p[l] * mu[i];            /* l in C_{n+1}^m, mu_lm = nu_i    */
                    }
                    double den = state_lambda(&R, m) + state_mu(&R, m);
                    a[m] = up_in / (lam_prev * den);
                    b[m] = ratio * down_in / den;
                }
            }
            /* inner r-loop on the scalar mu^{k,r}(n) (reading C1) */
            double sma = 0.0, smb = 0.0, amax = 0.0;
            for (uint64_t t = 0; t < c; t++) {
                uint64_t m = L[t];
                double mm = state_mu(&R, m);
                sma += mm * a[m];
                smb += mm * b[m];
                if (a[m] > amax) amax = a[m];
            }
            double muk = mu_n[n];   /* mu^{k,0}(n) = mu^{k-1}(n) */
            double prev_dp = INFINITY;
            for (int r = 0; r < 100000; r++) {
                double nxt = muk * sma + smb;   /* Eq. muHeter applied to Eq. updateHeter */
                double dp = fabs(nxt - muk) * amax;   /* max_m |p^{k,r} - p^{k,r-1}| */
                muk = nxt;
                if (dp == 0.0 || dp >= prev_dp) break;   /* no further change at fp64 */
                prev_dp = dp;
            }
            /* p_n^k = mu^k a + b, then renormalise (reading C2) */
            double sp = 0.0;
            for (uint64_t t = 0; t < c; t++) {
                uint64_t m = L[t];
                p[m] = muk * a[m] + b[m];
                sp += p[m];
            }
            double sl = 0.0, sm = 0.0;
            for (uint64_t t = 0; t < c; t++) {
                uint64_t m = L[t];
                p[m] /= sp;
                sl += p[m] * state_lambda(&R, m);
                sm += p[m] * state_mu(&R, m);
            }
            lam_n[n] = sl;   /* Eq. lambdaHeter */
            mu_n[n] = sm;    /* Eq. muHeter     */
        }
        /* Proposition 1 + Eq. bnd_stationary */
        birth_death(N, lam_n, mu_n, pn);
#pragma omp parallel for schedule(static)
        for (int64_t m = 0; m < (int64_t)S; m++) pi_out[m] = pn[popcount64((uint64_t)m)] * p[m];
        res = residual(&R, pi_out);
        if (trace) trace[k - 1] = res;
        if (!(res == res)) { status = ORACLE_E_INVAL; break; }
        if (res <= tol) { status = ORACLE_OK; break; }
    }
    if (iters_out) *iters_out = k;
    if (residual_out) *residual_out = res;
    if (layer_lam_out) memcpy(layer_lam_out, lam_n, sizeof(double) * (N + 1));
    if (layer_mu_out) memcpy(layer_mu_out, mu_n, sizeof(double) * (N + 1));

    for (int n = 0; n <= N; n++) free(lay[n]);
    free(lay); free(cnt); free(p); free(a); free(b); free(lam_n); free(mu_n); free(pn);
    free(R.Wtab); free(R.lamtab); free(R.mutab);
    return status;
}

double oracle_residual(int N, int J, const double *lam, const double *mu, const int32_t *pref, const double *pi) {
    inst_t I = {N, J, lam, mu, pref};
    rates_t R = {&I, NULL, NULL, NULL};
    return residual(&R, pi);
}

/* ---------------------------------------------------------------------- */
/* Memory-lean residual (full-size checks)                                 */
/* ---------------------------------------------------------------------- */

/* Prefix tree of the preference lists: one node per distinct list prefix
 * zeta_j(1..h); thr[v] = sum of lam_j over the atoms whose list starts with
 * that prefix.  Children are kept as a first-child / next-sibling list. */
typedef struct {
    int n, cap;
    int *unit, *child, *sib;
    double *thr;
} ptree_t;

static int ptree_node(ptree_t *T, int unit) {
    if (T->n == T->cap) {
        T->cap = T->cap ? 2 * T->cap : 1024;
        T->unit = (int *)realloc(T->unit, sizeof(int) * T->cap);
        T->child = (int *)realloc(T->child, sizeof(int) * T->cap);
        T->sib = (int *)realloc(T->sib, sizeof(int) * T->cap);
        T->thr = (double *)realloc(T->thr, sizeof(double) * T->cap);
    }
    T->unit[T->n] = unit;
    T->child[T->n] = -1;
    T->sib[T->n] = -1;
    T->thr[T->n] = 0.0;
    return T->n++;
}

static void ptree_build(const inst_t *I, ptree_t *T) {
    memset(T, 0, sizeof(*T));
    ptree_node(T, -1);   /* root: the empty prefix */
    for (int j = 0; j < I->J; j++) {
        int cur = 0;
        for (int h = 0; h < I->N; h++) {
            int u = I->pref[(size_t)j * I->N + h];
            if (u < 0) break;
            int c = T->child[cur];
            while (c >= 0 && T->unit[c] != u) c = T->sib[c];
            if (c < 0) {
                c = ptree_node(T, u);
                T->sib[c] = T->child[cur];
                T->child[cur] = c;
            }
            T->thr[c] += I->lam[j];
            cur = c;
        }
    }
}

static void ptree_free(ptree_t *T) { free(T->unit); free(T->child); free(T->sib); free(T->thr); }

/* Eq. tran_rates at state m through the prefix tree (readings C6, C19): the
 * atoms through a node whose units are all busy in m reach its children; a
 * child whose unit i is busy receives them as the upward rate W[i] =
 * lambda_{m\i -> m}; a free child's unit is their first free unit, so they
 * count in lambda_m; atoms whose whole list is busy are lost (C = 0). */
static double ptree_rates(const ptree_t *T, int N, uint64_t m, double *W, int *stk) {
    for (int i = 0; i < N; i++) W[i] = 0.0;
    double lm = 0.0;
    int sp = 0;
    stk[sp++] = 0;
    while (sp > 0) {
        int v = stk[--sp];
        for (int c = T->child[v]; c >= 0; c = T->sib[c]) {
            int u = T->unit[c];
            if ((m >> u) & 1) {
                W[u] += T->thr[c];
                stk[sp++] = c;
            } else {
                lm += T->thr[c];
            }
        }
    }
    return lm;
}

/*
 * The relative L1 global-balance residual r(pi) of Eq. balance_eq_heter
 * (reading C3) with O(2^(N - block_bits)) scratch: the rates
 * of each state come from the prefix tree (ptree_rates), per-state terms are
 * summed in ascending state order inside blocks of 2^block_bits states and the
 * block sums in ascending block order.  num_out / den_out receive the two sums.
 */
double oracle_residual_stream(int N, int J, const double *lam, const double *mu, const int32_t *pref,
                              const double *pi, int block_bits, double *num_out, double *den_out) {
    inst_t I = {N, J, lam, mu, pref};
    ptree_t T;
    ptree_build(&I, &T);
    if (block_bits > N) block_bits = N;
    if (block_bits < 0) block_bits = 0;
    const uint64_t nb = 1ULL << (N - block_bits), bs = 1ULL << block_bits;
    double *bnum = (double *)malloc(sizeof(double) * nb), *bden = (double *)malloc(sizeof(double) * nb);
    if (!bnum || !bden) { free(bnum); free(bden); ptree_free(&T); return NAN; }
#pragma omp parallel
    {
        double W[64];
        int *stk = (int *)malloc(sizeof(int) * (T.n + 1));
#pragma omp for schedule(dynamic, 16)
        for (int64_t b = 0; b < (int64_t)nb; b++) {
            double sn = 0.0, sd = 0.0;
            for (uint64_t k = 0; k < bs; k++) {
                uint64_t m = ((uint64_t)b << block_bits) | k;
                double lm = ptree_rates(&T, N, m, W, stk);
                double out = pi[m] * (lm + mu_m(&I, m));
                double in = 0.0;
                for (int i = 0; i < N; i++) {
                    uint64_t l = m ^ (1ULL << i);
                    if ((m >> i) & 1) in += pi[l] * W[i];   /* upward transition into m   */
                    else in += pi[l] * mu[i];                /* downward transition into m */
                }
                sn += fabs(out - in);
                sd += out;
            }
            bnum[b] = sn;
            bden[b] = sd;
        }
        free(stk);
    }
    double num = 0.0, den = 0.0;
    for (uint64_t b = 0; b < nb; b++) { num += bnum[b]; den += bden[b]; }
    free(bnum); free(bden); ptree_free(&T);
    if (num_out) *num_out = num;
    if (den_out) *den_out = den;
    return num / den;
}

/* Eq. tran_rates through the prefix tree at one state (tests: equals
 * oracle_dispatch_rates / lambda_m by list scans).  Returns lambda_m. */
double oracle_tree_rates(int N, int J, const double *lam, const int32_t *pref, uint64_t m, double *W) {
    inst_t I = {N, J, lam, NULL, pref};
    ptree_t T;
    ptree_build(&I, &T);
    int *stk = (int *)malloc(sizeof(int) * (T.n + 1));
    double lm = ptree_rates(&T, N, m, W, stk);
    free(stk);
    ptree_free(&T);
    return lm;
}

double oracle_lambda_m(int N, int J, const double *lam, const int32_t *pref, uint64_t m) {
    inst_t I = {N, J, lam, NULL, pref};
    return lambda_m(&I, m);
}

/*
 * Balance of Eq. balance_eq_heter at individual states (for sampled checks).
 * nbr[s*(N+1) + 0] = pi(m_s), nbr[s*(N+1) + 1 + i] = pi(m_s xor 2^i).
 * out[2*s] = pi(m)(lambda_m+mu_m) (outflow), out[2*s+1] = inflow.
 */
int oracle_state_balance(int N, int J, const double *lam, const double *mu, const int32_t *pref,
                         const uint64_t *states, int64_t ns, const double *nbr, double *out) {
    inst_t I = {N, J, lam, mu, pref};
#pragma omp parallel
    {
        double W[64];
#pragma omp for schedule(static)
        for (int64_t s = 0; s < ns; s++) {
            uint64_t m = states[s];
            const double *v = nbr + (size_t)s * (N + 1);
            dispatch_rates(&I, m, W);
            double o = v[0] * (lambda_m(&I, m) + mu_m(&I, m));
            double in = 0.0;
            for (int i = 0; i < N; i++) {
                if ((m >> i) & 1) in += v[1 + i] * W[i];
                else in += v[1 + i] * mu[i];
            }
            out[2 * s] = o;
            out[2 * s + 1] = in;
        }
    }
    return ORACLE_OK;
}

/*
 * Performance measures by definition, by direct loops over states and atoms.
 *   workload[i] = rho_i = sum_{m: unit i busy} P{B_m}        (C12)
 *   for every state m and atom j: the dispatched unit is the first free unit
 *   of zeta_j (the sets S_ij); disp[j*N+i] accumulates
 *   f_j P{B_m}; if none is free the call is lost and loss += f_j P{B_m}.
 *   dispatch rho_ij = disp / (1 - loss) (reading C13: the
 *   fraction of served calls; for full lists loss = Pi = P{all busy}).
 * dispatch is returned row-major [j][i].
 */
int oracle_measures(int N, int J, const double *lam, const double *mu, const int32_t *pref, const double *pi,
                    double *workload, double *dispatch, double *loss_out) {
    (void)mu;
    uint64_t S = 1ULL << N;
    double Lam = 0.0;
    for (int j = 0; j < J; j++) Lam += lam[j];
    for (int i = 0; i < N; i++) workload[i] = 0.0;
    for (int64_t q = 0; q < (int64_t)J * N; q++) dispatch[q] = 0.0;
    double loss = 0.0;
    for (uint64_t m = 0; m < S; m++) {
        double pm = pi[m];
        for (int i = 0; i < N; i++)
            if ((m >> i) & 1) workload[i] += pm;
        for (int j = 0; j < J; j++) {
            double fj = lam[j] / Lam;
            int found = -1;
            for (int h = 0; h < N; h++) {
                int u = pref[(size_t)j * N + h];
                if (u < 0) break;
                if (!((m >> u) & 1)) { found = u; break; }
            }
            if (found >= 0) dispatch[(size_t)j * N + found] += fj * pm;
            else loss += fj * pm;
        }
    }
    for (int64_t q = 0; q < (int64_t)J * N; q++) dispatch[q] /= (1.0 - loss);
    *loss_out = loss;
    return ORACLE_OK;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
