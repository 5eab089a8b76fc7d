// hq_api.cu -- host orchestration behind the C-ABI declared in include/hq.h.
//
// hq_create validates the instance and builds the
// preference trie used by the kernels to evaluate the upward transition rates
// of Eq. tran_rates on the fly.  hq_solve runs the
// red-black staggered schedule of Algorithm 1 (DESIGN.md
// §2): half-sweep t updates every layer n = t (mod 2), 1 <= n <= min(t, N-1),
// from the current layers n-1 and n+1.  Layer n at half-sweep t performs its
// k-th update, k = (t-n)/2 + 1, and reads layer n-1 at its k-th update and
// layer n+1 at its (k-1)-th: exactly the data dependencies of Alg. 1's
// sequential layer loop, so the iterates equal
// Algorithm 1's up to floating-point rounding.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hq.h"
#include "hq_internal.h"
#include "hq_v2.h"
#include "hq_v3.h"

// ---- device memory: the CUDA default memory pool (stream-ordered allocator), so that the
// working set of a handle is recycled across handles without page (un)mapping; blocks above
// the release threshold go back to the driver at the next synchronisation.  dfree keeps
// cudaFree's device-wide synchronisation (nothing may still use the block).
void hq_pool_init() {   // also used by hq_batch.cu
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = 8ull << 30;   // keep up to 8 GB cached between handles
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
    });
}
static cudaError_t dmalloc(void **p, size_t bytes) {
    hq_pool_init();
    cudaError_t e = cudaMallocAsync(p, bytes ? bytes : 16, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);   // usable from any stream on return
    if (e != cudaSuccess) {
        *p = nullptr;
        cudaGetLastError();
    }
    return e;
}
static void dfree(void *p) {
    if (!p) return;
    cudaDeviceSynchronize();
    cudaFreeAsync(p, 0);
}
// small pinned host buffers, recycled across handles (cudaMallocHost / cudaFreeHost are slow)
static std::mutex g_pin_mu;
static std::vector<std::pair<size_t, void *>> g_pin_free;
static cudaError_t pinned_alloc(void **p, size_t bytes) {
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        for (size_t i = 0; i < g_pin_free.size(); i++)
            if (g_pin_free[i].first == bytes) {
                *p = g_pin_free[i].second;
                g_pin_free.erase(g_pin_free.begin() + (long)i);
                return cudaSuccess;
            }
    }
    return cudaMallocHost(p, bytes);
}
static void pinned_free(void *p, size_t bytes) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    if (g_pin_free.size() < 64) g_pin_free.emplace_back(bytes, p);
    else cudaFreeHost(p);
}

namespace hqk_launch {
cudaError_t gather(const KArgs &k, int grid, cudaStream_t s);
cudaError_t finalize(const KArgs &k, int grid, cudaStream_t s);
cudaError_t init(const KArgs &k, int grid, cudaStream_t s);
cudaError_t residual(const KArgs &k, int grid, cudaStream_t s);
cudaError_t layer_reduce(int N, uint32_t active, int ncta, int nbuf, const double *partial, int NV, int mode,
                         double *lam_n, double *mu_n, double *mustar, double *stats, int *err, cudaStream_t s);
cudaError_t assemble(int N, const double *pw, const double *pn, double *pi, int grid, cudaStream_t s);
cudaError_t zeta(int N, double *g, int grid, cudaStream_t s);
cudaError_t measures(int N, int J, const double *lam, double Lam, const int32_t *pref, const double *g,
                     double *workload, double *dispatch, double *loss, cudaStream_t s);
cudaError_t scale(double *x, uint64_t n, double f, int grid, cudaStream_t s);
cudaError_t response(int N, int J, const double *lam, double Lam, const double *disp, const double *tau, double T,
                     double *mrt_j, double *f_j, double *tot, cudaStream_t s);
cudaError_t buffer_measures(int N, int J, const double *lam, double Lam, const double *nu, const double *pi_all_busy,
                            const double *loss_dev, double tail_mass, double tail_last, double loss_q,
                            double *workload, double *dispatch, cudaStream_t s);
int tile_states();
cudaError_t init_v2(const KArgs &k, int grid, cudaStream_t s);
}  // namespace hqk_launch

// internal status (never returned by the ABI): an instance whose rate programs do not fit the
// tiled paths' format; hq_solve falls back to path 1 (per-thread trie walk, any instance)
static const hq_status HQ_I_OVERFLOW = (hq_status)-100;

namespace {

thread_local std::string g_create_error;

struct TrieHost {
    std::vector<int2> node;
    std::vector<double> lam_thr, lam_end;
};

// Preference trie: one node per distinct list prefix; Lambda_v = sum of
// lambda_j over atoms whose list passes through v; lam_end = atoms whose
// (truncated) list ends at v.  Emitted in preorder with skip indices.
TrieHost build_trie(int N, int J, const double *lam, const int32_t *pref) {
    struct TN {
        int unit;
        double thr = 0.0, end = 0.0;
        std::map<int, int> child;
    };
    std::vector<TN> t(1);
    t[0].unit = -1;
    for (int j = 0; j < J; j++) {
        if (!(lam[j] > 0.0)) continue;
        int cur = 0;
        int last = -1;
        for (int h = 0; h < N; h++) {
            const int u = pref[(size_t)j * N + h];
            if (u < 0) break;
            auto it = t[cur].child.find(u);
            int nx;
            if (it == t[cur].child.end()) {
                nx = (int)t.size();
                t[cur].child[u] = nx;
                TN c;
                c.unit = u;
                t.push_back(c);
            } else {
                nx = it->second;
            }
            t[nx].thr += lam[j];
            cur = nx;
            last = nx;
        }
        if (last >= 0) t[last].end += lam[j];
    }
    TrieHost out;
    // iterative preorder over the children of the root
    std::vector<int> order;
    std::vector<int> pre_of(t.size(), -1);
    std::vector<int> stk;
    for (auto it = t[0].child.rbegin(); it != t[0].child.rend(); ++it) stk.push_back(it->second);
    while (!stk.empty()) {
        int v = stk.back();
        stk.pop_back();
        pre_of[v] = (int)order.size();
        order.push_back(v);
        for (auto it = t[v].child.rbegin(); it != t[v].child.rend(); ++it) stk.push_back(it->second);
    }
    const int nn = (int)order.size();
    // subtree sizes for skip indices
    std::vector<int> size(t.size(), 1);
    for (int p = nn - 1; p >= 0; p--) {
        const int v = order[p];
        for (auto &kv : t[v].child) size[v] += size[kv.second];
    }
    std::vector<int> depth(t.size(), 0);
    for (int p = 0; p < nn; p++) {
        const int v = order[p];
        for (auto &kv : t[v].child) depth[kv.second] = depth[v] + 1;
    }
    for (auto &kv : t[0].child) depth[kv.second] = 1;
    for (int p = 0; p < nn; p++) {
        const int v = order[p];
        for (auto &kv : t[v].child) depth[kv.second] = depth[v] + 1;
    }
    out.node.resize(nn);
    out.lam_thr.resize(nn);
    out.lam_end.resize(nn);
    for (int p = 0; p < nn; p++) {
        const int v = order[p];
        out.node[p] = make_int2(t[v].unit | (depth[v] << 8), p + size[v]);
        out.lam_thr[p] = t[v].thr;
        out.lam_end[p] = t[v].end;
    }
    return out;
}

double binom(int n, int k) {
    if (k < 0 || k > n) return 0.0;
    double r = 1.0;
    for (int i = 1; i <= k; i++) r = r * (double)(n - k + i) / (double)i;
    return std::floor(r + 0.5);
}



// Internal unit order for the CTA-tiled path (hq_v3.h).  Rate programs are per warp
// tile: only units 0 (parity), 1, 7, 8 (register bits) and 2..6 (lanes) vary inside a
// program; every other unit is fixed per program and its trie nodes fold into the
// warp-tile-uniform rates.  So the nine units that least often precede other units in the
// preference lists vary, and among them the four register-class slots (whose pairs need
// per-state masks, the expensive "groups") go to the units that minimise the expected
// number of register-dependent nodes alive in a random warp tile.  Warp and tile units
// follow in order of increasing prefix count.
std::vector<int> choose_perm_v3(int N, const TrieHost &tr, int nW) {
    (void)nW;
    std::vector<int> perm(N);
    for (int u = 0; u < N; u++) perm[u] = u;
    const char *env = getenv("HQ_PERM");
    if (env && std::string(env) == "identity") return perm;
    std::vector<long> cnt(N, 0);
    std::vector<int> stk;
    std::vector<uint32_t> pre(tr.node.size()), pstk;
    for (size_t v = 0; v < tr.node.size(); v++) {
        const int u = tr.node[v].x & 0xff, d = (tr.node[v].x >> 8) & 0xff;
        stk.resize(d - 1);
        pstk.resize(d - 1);
        for (int a : stk) cnt[a]++;
        pre[v] = d >= 2 ? pstk[d - 2] : 0u;
        stk.push_back(u);
        pstk.push_back(pre[v] | (1u << u));
    }
    std::vector<int> idx(N);
    for (int u = 0; u < N; u++) idx[u] = u;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return cnt[a] < cnt[b]; });
    std::vector<int> V(idx.begin(), idx.begin() + 9);
    uint32_t vmask = 0;
    for (int x : V) vmask |= 1u << x;
    // node weight: probability that its fixed-unit path is busy in a random warp tile
    std::vector<double> w(tr.node.size());
    for (size_t v = 0; v < tr.node.size(); v++) {
        const int u = tr.node[v].x & 0xff;
        w[v] = std::ldexp(1.0, -__builtin_popcount((pre[v] | (1u << u)) & ~vmask));
    }
    double best = 1e300;
    uint32_t bestT = 0;
    for (int a1 = 0; a1 < 9; a1++)
        for (int a2 = a1 + 1; a2 < 9; a2++)
            for (int a3 = a2 + 1; a3 < 9; a3++)
                for (int a4 = a3 + 1; a4 < 9; a4++) {
                    const uint32_t T = (1u << V[a1]) | (1u << V[a2]) | (1u << V[a3]) | (1u << V[a4]);
                    double cost = 0.0;
                    for (size_t v = 0; v < tr.node.size(); v++)
                        if (pre[v] & T) cost += w[v];
                    if (cost < best) {
                        best = cost;
                        bestT = T;
                    }
                }
    std::vector<int> regc, rest;
    for (int x : V) ((bestT >> x) & 1u ? regc : rest).push_back(x);
    perm[0] = regc[0];
    perm[1] = regc[1];
    perm[7] = regc[2];
    perm[8] = regc[3];
    for (int u = 2; u <= 6; u++) perm[u] = rest[u - 2];
    for (int q = 9; q < N; q++) perm[q] = idx[q];
    return perm;
}
}  // namespace

enum { S_LAM = 0, S_MU = 32, S_MUSTAR = 64, S_PN = 96, S_STATS = 128, S_INVC = 256, S_TOTAL = 288 };

struct hq_problem {
    int N = 0, J = 0;
    double Lam = 0.0;
    bool full_lists = true;
    std::vector<double> lam, mu;
    std::vector<int32_t> pref;
    TrieHost trie;                 // internal unit ids
    std::vector<int> perm;         // internal unit -> ABI unit
    std::vector<double> nu_int;    // service rates in internal order
    std::string err;
    int device = -1;
    bool dev_ready = false;        // every per-device buffer of `device` allocated and filled
    int nsm = 0;
    bool solved = false;
    // waiting room (hq_set_buffer): 0 loss system, C > 0 finite buffer, -1 unlimited
    int bufC = 0;
    cudaStream_t side = nullptr;   // path 3 precompute: scatter weights beside the rate programs
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    double q_r = 0.0;        // Lambda / sum nu
    double q_first = 0.0;    // P~{1} of the last solve
    double q_mass = 0.0;     // sum_c P~{c}
    double q_last = 0.0;     // P~{C} (finite C), 0 for an unlimited buffer
    double stats[HQ_STATS_LEN] = {0};
    // device memory
    bool dev_loop = true;          // path 3: device-resident solve (k_loop3); HQ_LOOP=host: one launch per half-sweep
    Ctl3 *d_ctl = nullptr, *h_ctl = nullptr;   // path 3, device loop: control block (+ pinned mirror)
    unsigned long long *d_xg = nullptr;        // path 3, device loop: exact phase sums
    int2 *d_node = nullptr;
    double *d_lthr = nullptr, *d_lend = nullptr;
    double *d_lam = nullptr;
    int32_t *d_pref = nullptr;
    double *d_pw = nullptr;        // [2^N] conditional probabilities, parity-compressed
    double2 *d_ab = nullptr;       // [2^(N-1)] (a,b) scratch; also superset-sum scratch
    double *d_partial = nullptr;   // [2][grid][HQ_NL][HQ_NV]
    double *d_small = nullptr;     // lam_n, mu_n, mustar, pn, stats, invC
    int *d_err = nullptr;
    double *h_small = nullptr;     // pinned mirror
    int grid = 0;
    // v2 (N >= 8) device state
    bool v2 = false, v2_ready = false;
    int path = 1;                  // 1: N < 9 two-pass (hq_kernels.cu), 3: CTA-tiled (hq_v3.cu)
    int nW = 0;                    // path 3: log2(warps per CTA)
    uint32_t maxblk_all = 0;       // path 3: largest program block of a CTA tile (records)
    unsigned long long *d_wtime = nullptr;   // path 3: per-warp busy cycles (-DHQ_WARP_TIMING builds)
    int prog_nwv = 0;              // path 3: warp bits varying inside a rate program (nW: CTA programs)
    bool chunked = false;          // path 3: chunked tile order (else popcount order)
    int chunk_bits = 0;            // path 3, chunked order: low tile bits per chunk
    int h_in = 32;                 // path 3: tile-unit neighbours h < h_in are loaded evict-last
    int h_out_pol = 0;             // path 3: L2 policy of the other tile-unit neighbour loads
    int pf_h = 0, pf_o = 0;        // path 3: L2 prefetch distance of the tile-unit slices; of omega/kappa
    int in_pol = 0;                // path 3: L2 policy of the q blocks and in-group neighbours (S3Args::pol)
    int pf_min = 0;                // path 3: prefetch only the tile units h >= pf_min
    // path 3, group order: group progress bound (S3Args::gs_ctr); gs_lag 0 = off
    int gs_lag = 0;
    uint32_t gs_ng = 0;
    unsigned long long *d_gsctr = nullptr, gs_epoch = 0;
    std::vector<uint32_t> chunk_range;   // path 3, chunked order: CTA ranges over the visit order
    uint32_t *d_order = nullptr, *d_off16 = nullptr, *d_size16 = nullptr, *d_range = nullptr;
    uint4 *d_prog = nullptr;
    double2 *d_omkap = nullptr;
    double *d_lamarr = nullptr;
    double *d_blk = nullptr, *h_blk = nullptr;
    int sgrid = 0;
    uint32_t total16 = 0, maxrec = 0;
    double prog_bytes = 0.0, precompute_ms = 0.0;
    std::vector<cudaEvent_t> ev;   // per-half-sweep timing events (pairs), reused across solves

    cudaEvent_t event(size_t i) {
        while (ev.size() <= i) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            ev.push_back(e);
        }
        return ev[i];
    }

    ~hq_problem() { release(); }
    void release() {
        dfree(d_node);
        dfree(d_lthr);
        dfree(d_lend);
        dfree(d_lam);
        dfree(d_pref);
        dfree(d_pw);
        dfree(d_ab);
        dfree(d_partial);
        dfree(d_small);
        dfree(d_err);
        dfree(d_order);
        dfree(d_range);
        d_range = nullptr;
        dfree(d_wtime);
        d_wtime = nullptr;
        dfree(d_gsctr);
        d_gsctr = nullptr;
        gs_epoch = 0;
        dfree(d_off16);
        dfree(d_size16);
        dfree(d_prog);
        dfree(d_omkap);
        dfree(d_lamarr);
        dfree(d_blk);
        dfree(d_ctl);
        dfree(d_xg);
        pinned_free(h_ctl, sizeof(Ctl3));
        d_ctl = h_ctl = nullptr;
        d_xg = nullptr;
        if (side) cudaStreamDestroy(side);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        side = nullptr;
        ev_fork = ev_join = nullptr;
        for (auto e : ev) cudaEventDestroy(e);   // events belong to the device they were created on
        ev.clear();
        pinned_free(h_blk, sizeof(double) * V2S_TOTAL);
        d_order = d_off16 = d_size16 = nullptr;
        d_prog = nullptr;
        d_omkap = nullptr;
        d_lamarr = d_blk = h_blk = nullptr;
        v2_ready = false;
        dev_ready = false;
        pinned_free(h_small, sizeof(double) * S_TOTAL);
        d_node = nullptr;
        d_lthr = d_lend = d_lam = nullptr;
        d_pref = nullptr;
        d_pw = nullptr;
        d_ab = nullptr;
        d_partial = d_small = nullptr;
        d_err = nullptr;
        h_small = nullptr;
    }
};

// small-array layout inside d_small / h_small

#define HQ_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t e__ = (call);                                                       \
        if (e__ != cudaSuccess) {                                                       \
            h->err = std::string("CUDA error: ") + cudaGetErrorString(e__) + " at " #call; \
            return HQ_E_CUDA;                                                           \
        }                                                                               \
    } while (0)

static hq_status fail_create(const std::string &msg) {
    g_create_error = msg;
    return HQ_E_INVAL;
}

extern "C" hq_status hq_create(int N, int J, const double *lambda, const double *mu, const int32_t *pref,
                               hq_handle *out) {
    if (!out) return fail_create("out is NULL");
    *out = nullptr;
    if (N < 1 || N > HQ_MAXN) return fail_create("N must be in [1, 31]");
    if (J < 1) return fail_create("J must be >= 1");
    if (!lambda || !mu || !pref) return fail_create("NULL input array");
    double Lam = 0.0;
    for (int j = 0; j < J; j++) {
        if (!std::isfinite(lambda[j]) || lambda[j] < 0.0) return fail_create("lambda[j] must be finite and >= 0");
        Lam += lambda[j];
    }
    if (!(Lam > 0.0)) return fail_create("sum of lambda must be > 0");
    for (int i = 0; i < N; i++)
        if (!std::isfinite(mu[i]) || !(mu[i] > 0.0)) return fail_create("mu[i] must be finite and > 0");
    bool full = true;
    std::vector<char> reach(N, 0);
    for (int j = 0; j < J; j++) {
        std::vector<char> seen(N, 0);
        bool ended = false;
        int len = 0;
        for (int h = 0; h < N; h++) {
            const int u = pref[(size_t)j * N + h];
            if (u == -1) {
                ended = true;
                continue;
            }
            if (ended) return fail_create("pref row " + std::to_string(j) + ": entry after -1 padding");
            if (u < 0 || u >= N) return fail_create("pref row " + std::to_string(j) + ": unit id out of range");
            if (seen[u]) return fail_create("pref row " + std::to_string(j) + ": duplicated unit");
            seen[u] = 1;
            len++;
            if (lambda[j] > 0.0) reach[u] = 1;
        }
        if (len == 0) return fail_create("pref row " + std::to_string(j) + " is empty");
        if (len < N) full = false;
    }
    for (int i = 0; i < N; i++)
        if (!reach[i])
            return fail_create("unit " + std::to_string(i) +
                               " is in no list of an atom with lambda > 0 (reducible chain)");

    auto h = std::make_unique<hq_problem>();
    h->N = N;
    h->J = J;
    h->Lam = Lam;
    h->full_lists = full;
    h->lam.assign(lambda, lambda + J);
    h->mu.assign(mu, mu + N);
    h->pref.assign(pref, pref + (size_t)J * N);
    {
        TrieHost abi = build_trie(N, J, lambda, pref);
        // N < 9: the two-pass kernels (per-thread trie walk); N >= 9: the CTA-tiled path
        h->path = N < 9 ? 1 : 3;
        if (h->path == 3) {
            h->nW = hq3_launch::choose_nw(N);
            if (const char *wenv = getenv("HQ_NW"))   // development override (log2 warps per CTA)
                h->nW = std::max(0, std::min({atoi(wenv), 4, N - 9}));
            h->perm = choose_perm_v3(N, abi, h->nW);
        } else {   // the two-pass path works in ABI unit order
            h->perm.resize(N);
            for (int u = 0; u < N; u++) h->perm[u] = u;
        }
        std::vector<int> inv(N);
        for (int u = 0; u < N; u++) inv[h->perm[u]] = u;
        std::vector<int32_t> pint((size_t)J * N);
        for (size_t q = 0; q < pint.size(); q++) pint[q] = pref[q] < 0 ? -1 : inv[pref[q]];
        h->trie = build_trie(N, J, lambda, pint.data());
        h->nu_int.resize(N);
        for (int u = 0; u < N; u++) h->nu_int[u] = mu[h->perm[u]];
    }
    h->v2 = h->path == 3;   // the tiled path (a-priori normalisation, one pass per half-sweep)
    // device-resident solve by default where it is the faster path (measured, DESIGN.md §9:
    // N = 18 14.3 vs 16.2 ms; N = 24 145 vs 123 ms); HQ_LOOP=device|host overrides
    h->dev_loop = N < 21;
    if (const char *lenv = getenv("HQ_LOOP")) h->dev_loop = std::string(lenv) != "host";
    *out = h.release();
    return HQ_OK;
}

static hq_status alloc_device(hq_problem *h);

static hq_status ensure_device(hq_problem *h) {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        h->err = std::string("no CUDA device: ") + cudaGetErrorString(e);
        return HQ_E_CUDA;
    }
    if (h->device == dev && h->dev_ready) return HQ_OK;
    if (h->device != -1) h->release();   // other device, or a partial set from a failed call
    h->device = dev;
    const hq_status st = alloc_device(h);
    if (st != HQ_OK) {   // never keep a partial buffer set: the next call starts over
        cudaGetLastError();
        h->release();
        h->device = -1;
        return st;
    }
    h->dev_ready = true;
    return HQ_OK;
}

static hq_status alloc_device(hq_problem *h) {
    const int dev = h->device;
    HQ_CUDA(cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, dev));
    const int N = h->N;
    const size_t S = (size_t)1 << N;
    const uint64_t ntiles = ((S >> 1) + hqk_launch::tile_states() - 1) / hqk_launch::tile_states();
    h->grid = (int)std::min<uint64_t>(ntiles, (uint64_t)h->nsm * 4);
    const size_t nn = h->trie.node.size();
    auto alloc = [&](void **p, size_t bytes) -> cudaError_t { return dmalloc(p, bytes ? bytes : 16); };
    if (h->path == 3) {
        // host loop: a grid of CTAs in waves; device loop: one co-resident CTA per SM
        const uint64_t nt3 = 1ull << (N - 9 - h->nW);
        const int per_sm = h->dev_loop ? 1 : hq3_launch::ctas_per_sm(h->nW);
        h->sgrid = (int)std::min<uint64_t>(nt3, (uint64_t)h->nsm * per_sm);
    } else {
        h->sgrid = hq2_launch::sweep_grid(h->nsm);
    }
    if (alloc((void **)&h->d_pw, sizeof(double) * S) != cudaSuccess ||
        (!h->v2 && alloc((void **)&h->d_ab, sizeof(double2) * (S >> 1 ? S >> 1 : 1)) != cudaSuccess) ||
        (h->v2 && alloc((void **)&h->d_omkap, sizeof(double2) * S) != cudaSuccess)) {
        h->err = "device memory for the working set (2^N doubles x 2) could not be allocated";
        return HQ_E_NOMEM;
    }
    HQ_CUDA(alloc((void **)&h->d_node, sizeof(int2) * nn));
    HQ_CUDA(alloc((void **)&h->d_lthr, sizeof(double) * nn));
    HQ_CUDA(alloc((void **)&h->d_lend, sizeof(double) * nn));
    HQ_CUDA(alloc((void **)&h->d_lam, sizeof(double) * h->J));
    HQ_CUDA(alloc((void **)&h->d_pref, sizeof(int32_t) * h->J * N));
    HQ_CUDA(alloc((void **)&h->d_partial, sizeof(double) * 2 * std::max(h->grid, h->sgrid) * HQ_NL * HQ_NV));
    HQ_CUDA(alloc((void **)&h->d_blk, sizeof(double) * 2 * V2S_TOTAL));   // [0]: the block, [1]: fold buffer
    HQ_CUDA(pinned_alloc((void **)&h->h_blk, sizeof(double) * V2S_TOTAL));
    HQ_CUDA(alloc((void **)&h->d_small, sizeof(double) * S_TOTAL));
    HQ_CUDA(alloc((void **)&h->d_err, sizeof(int)));
    HQ_CUDA(pinned_alloc((void **)&h->h_small, sizeof(double) * S_TOTAL));
    HQ_CUDA(cudaMemcpy(h->d_node, h->trie.node.data(), sizeof(int2) * nn, cudaMemcpyHostToDevice));
    HQ_CUDA(cudaMemcpy(h->d_lthr, h->trie.lam_thr.data(), sizeof(double) * nn, cudaMemcpyHostToDevice));
    HQ_CUDA(cudaMemcpy(h->d_lend, h->trie.lam_end.data(), sizeof(double) * nn, cudaMemcpyHostToDevice));
    HQ_CUDA(cudaMemcpy(h->d_lam, h->lam.data(), sizeof(double) * h->J, cudaMemcpyHostToDevice));
    HQ_CUDA(cudaMemcpy(h->d_pref, h->pref.data(), sizeof(int32_t) * h->J * N, cudaMemcpyHostToDevice));
    return HQ_OK;
}

static KArgs base_args(hq_problem *h) {
    KArgs k;
    memset(&k, 0, sizeof(k));
    k.N = h->N;
    k.full_lists = h->full_lists ? 1 : 0;
    k.nstates_c = (uint64_t)1 << (h->N - 1);
    k.ntiles = (k.nstates_c + hqk_launch::tile_states() - 1) / hqk_launch::tile_states();
    k.Lam = h->Lam;
    for (int i = 0; i < 32; i++) k.nu[i] = i < h->N ? h->nu_int[i] : 0.0;
    k.trie.nnodes = (int)h->trie.node.size();
    k.trie.node = h->d_node;
    k.trie.lam_thr = h->d_lthr;
    k.trie.lam_end = h->d_lend;
    k.ab = h->d_ab;
    k.lam_n = h->d_small + S_LAM;
    k.mu_n = h->d_small + S_MU;
    k.mustar = h->d_small + S_MUSTAR;
    k.pn = h->d_small + S_PN;
    return k;
}

static void class_arrays(hq_problem *h, KArgs &k, int c) {
    const size_t half = (size_t)1 << (h->N - 1);
    k.c = c;
    k.P = h->d_pw + (c ? half : 0);
    k.Q = h->d_pw + (c ? 0 : half);
}

// Eq. bnd_stationary on the host from the device layer rates.
static void birth_death(int N, const double *lam_n, const double *mu_n, double *pn) {
    double prod = 1.0, tot = 1.0;
    std::vector<double> g(N + 1);
    g[0] = 1.0;
    for (int n = 1; n <= N; n++) {
        prod *= lam_n[n - 1] / mu_n[n];
        g[n] = prod;
        tot += prod;
    }
    for (int n = 0; n < HQ_NL; n++) pn[n] = n <= N ? g[n] / tot : 0.0;
}

// True relative residual r(pi) of the current iterate; writes p(n) to device.
static hq_status true_residual(hq_problem *h, cudaStream_t s, double *res, int *launches) {
    const int N = h->N;
    double *hs = h->h_small;
    HQ_CUDA(cudaMemcpyAsync(hs, h->d_small, sizeof(double) * S_TOTAL, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    birth_death(N, hs + S_LAM, hs + S_MU, hs + S_PN);
    HQ_CUDA(cudaMemcpyAsync(h->d_small + S_PN, hs + S_PN, sizeof(double) * 32, cudaMemcpyHostToDevice, s));
    KArgs k = base_args(h);
    for (int c = 0; c < 2; c++) {
        class_arrays(h, k, c);
        k.partial = h->d_partial + (size_t)c * h->grid * HQ_NL * HQ_NV;
        HQ_CUDA(hqk_launch::residual(k, h->grid, s));
    }
    HQ_CUDA(hqk_launch::layer_reduce(N, 0, h->grid, 2, h->d_partial, 2, 3, nullptr, nullptr, nullptr,
                                     h->d_small + S_STATS, h->d_err, s));
    *launches += 3;
    HQ_CUDA(cudaMemcpyAsync(hs + S_STATS, h->d_small + S_STATS, sizeof(double) * 128, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    double num = 0.0, den = 0.0;
    for (int n = 0; n <= N; n++) {
        num += hs[S_STATS + n * 4 + 2];
        den += hs[S_STATS + n * 4 + 3];
    }
    *res = num / den;
    return HQ_OK;
}


// ---------------------------------------------------------------------------
// path 3 preparation: rate programs at warp-tile or CTA-tile granularity (hq_v3.h)
// ---------------------------------------------------------------------------
struct ProgSet {
    uint32_t *off16 = nullptr;   // [ntiles << nW] per-warp program offsets
    uint32_t *range = nullptr;   // [grid + 1] CTA tile ranges
    uint4 *prog = nullptr;
    uint32_t total16 = 0, maxblk = 0, cap = 0;
    int nwv = 0;
    void release() {
        dfree(off16);
        dfree(range);
        dfree(prog);
        off16 = range = nullptr;
        prog = nullptr;
    }
};

static hq_status v3_programs(hq_problem *h, cudaStream_t s, int nwv, const std::vector<uint32_t> &order,
                             ProgSet &ps) {
    const int N = h->N, nW = h->nW;
    const uint64_t ntiles = order.size(), W = 1ull << nW;
    const bool per_warp = (nwv == 0 && nW > 0);
    const uint64_t nprog = per_warp ? ntiles << nW : ntiles;
    std::vector<uint32_t> pord(nprog);
    for (uint64_t i = 0; i < ntiles; i++) {
        if (per_warp)
            for (uint64_t w = 0; w < W; w++) pord[(i << nW) | w] = (order[i] << nW) | (uint32_t)w;
        else
            pord[i] = order[i];
    }
    uint32_t *d_pord = nullptr, *d_size = nullptr, *d_offp = nullptr, *d_max = nullptr;
    void *tmp = nullptr;
    void *cache = nullptr;   // pair cache of the count pass (see below)
    auto cleanup = [&]() {
        dfree(d_pord);
        dfree(d_size);
        dfree(d_offp);
        dfree(d_max);
        dfree(tmp);
        dfree(cache);
        cache = nullptr;
    };
    if (dmalloc((void **)&d_pord, 4 * nprog) != cudaSuccess || dmalloc((void **)&d_size, 4 * nprog) != cudaSuccess ||
        dmalloc((void **)&d_offp, 4 * nprog) != cudaSuccess) {
        cudaGetLastError();
        cleanup();
        h->err = "device memory for the rate-program tables could not be allocated";
        return HQ_E_NOMEM;
    }
    HQ_CUDA(cudaMemcpyAsync(d_pord, pord.data(), 4 * nprog, cudaMemcpyHostToDevice, s));
    P3Args p3;
    memset(&p3, 0, sizeof(p3));
    p3.N = N;
    p3.nW = nW;
    p3.nwv = nwv;
    p3.full_lists = h->full_lists ? 1 : 0;
    p3.ntiles = nprog;
    for (int u = 0; u < 32; u++) p3.nu[u] = u < N ? h->nu_int[u] : 0.0;
    p3.nnodes = (int)h->trie.node.size();
    p3.node = h->d_node;
    p3.lam_thr = h->d_lthr;
    p3.lam_end = h->d_lend;
    const int g = h->nsm * 8;
    // pair cache for the write pass: a quarter of the free device memory (256 MB .. 2 GB),
    // at most 512 pairs per program
    {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
            cudaGetLastError();
            fr = 0;
        }
        const uint64_t budget = std::min<uint64_t>(2ull << 30, std::max<uint64_t>(256ull << 20, fr / 4));
        const int64_t per = (int64_t)(budget / nprog) - 32 * 8;
        const int ccap = (int)std::min<int64_t>(512, per > 0 ? per / 14 : 0);
        if (ccap >= 32 && dmalloc(&cache, nprog * ((size_t)ccap * 14 + 32 * 8 + 4)) == cudaSuccess) {
            char *c = static_cast<char *>(cache);
            p3.ccap = ccap;
            p3.cval = reinterpret_cast<double *>(c);
            c += nprog * (size_t)ccap * 8;
            p3.cW0 = reinterpret_cast<double *>(c);
            c += nprog * 32 * 8;
            p3.ckey = reinterpret_cast<uint32_t *>(c);
            c += nprog * (size_t)ccap * 4;
            p3.cn = reinterpret_cast<int *>(c);
            c += nprog * 4;
            p3.crm = reinterpret_cast<uint16_t *>(c);
        }
    }
    HQ_CUDA(cudaMemsetAsync(h->d_err, 0, sizeof(int), s));
    HQ_CUDA(hq3_launch::prog_count(p3, d_pord, d_size, h->d_err, g, s));
    size_t tb = 0;
    HQ_CUDA(hq2_launch::prog_scan(d_size, d_offp, nprog, nullptr, &tb, s));
    HQ_CUDA(dmalloc(&tmp, tb ? tb : 16));
    HQ_CUDA(hq2_launch::prog_scan(d_size, d_offp, nprog, tmp, &tb, s));
    std::vector<uint32_t> sz(nprog), offp(nprog);
    int herr = 0;
    HQ_CUDA(cudaMemcpyAsync(sz.data(), d_size, 4 * nprog, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaMemcpyAsync(offp.data(), d_offp, 4 * nprog, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaMemcpyAsync(&herr, h->d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    if (herr) {
        cleanup();
        h->err = "rate program overflow (too many distinct (unit, pattern) pairs in a tile)";
        return HQ_I_OVERFLOW;
    }
    const uint64_t total16 = (uint64_t)offp[nprog - 1] + sz[nprog - 1];
    if (total16 >= (1ull << 32)) {
        cleanup();
        h->err = "rate programs exceed 64 GB";
        return HQ_E_NOMEM;
    }
    ps.release();
    ps.nwv = nwv;
    ps.total16 = (uint32_t)total16;
    if (dmalloc((void **)&ps.prog, 16 * (total16 ? total16 : 1)) != cudaSuccess ||
        dmalloc((void **)&ps.off16, 4 * (ntiles << nW)) != cudaSuccess) {
        cudaGetLastError();
        cleanup();
        ps.release();
        h->err = "device memory for the rate programs could not be allocated";
        return HQ_E_NOMEM;
    }
    HQ_CUDA(hq3_launch::prog_write(p3, d_pord, d_offp, ps.prog, h->d_err, g, s));
    // per-warp program offsets (a CTA program serves every warp of its tile), block sizes,
    // work-balanced CTA ranges over the popcount-sorted tile order
    std::vector<uint32_t> off16(ntiles << nW);
    std::vector<double> cost(ntiles);
    double tot = 0.0;
    ps.maxblk = 0;
    for (uint64_t i = 0; i < ntiles; i++) {
        uint32_t b = 0, bmax = 0;
        for (uint64_t w = 0; w < W; w++) {
            off16[(i << nW) | w] = per_warp ? offp[(i << nW) | w] : offp[i];
            if (per_warp) {
                b += sz[(i << nW) | w];
                bmax = std::max(bmax, sz[(i << nW) | w]);
            }
        }
        if (!per_warp) b = bmax = sz[i];
        ps.maxblk = std::max(ps.maxblk, b);
        // estimated work of a tile in program-record units: the gather of its states plus
        // the evaluation of the program records (every warp evaluates a CTA program).  Chosen
        // by same-box A/B timing; models fitted to per-warp busy cycles balanced worse.
        cost[i] = 256.0 + (double)b * (per_warp ? 1.0 : (double)W / 4.0);

        tot += cost[i];
    }
    HQ_CUDA(cudaMemcpyAsync(ps.off16, off16.data(), 4 * off16.size(), cudaMemcpyHostToDevice, s));
    // optimal contiguous partition into G ranges (minimise the largest range cost): binary
    // search on the bottleneck with greedy packing
    const int G = h->sgrid;
    std::vector<uint32_t> range(G + 1, (uint32_t)ntiles);
    auto pack = [&](double cap, std::vector<uint32_t> *out) -> bool {
        int b = 0;
        double acc = 0.0;
        if (out) (*out)[0] = 0;
        for (uint64_t i = 0; i < ntiles; i++) {
            if (cost[i] > cap) return false;
            if (acc + cost[i] > cap) {
                if (++b >= G) return false;
                if (out) (*out)[b] = (uint32_t)i;
                acc = 0.0;
            }
            acc += cost[i];
        }
        if (out)
            for (int q = b + 1; q <= G; q++) (*out)[q] = (uint32_t)ntiles;
        return true;
    };
    double lo = tot / G, hi = tot;
    for (uint64_t i = 0; i < ntiles; i++) lo = std::max(lo, cost[i]);
    for (int it = 0; it < 60 && hi - lo > 1e-9 * hi; it++) {
        const double mid = 0.5 * (lo + hi);
        if (pack(mid, nullptr)) hi = mid;
        else lo = mid;
    }
    pack(hi, &range);
    if (h->chunked) range = h->chunk_range;   // chunked order: each CTA's own chunks
    HQ_CUDA(dmalloc((void **)&ps.range, 4 * (G + 1)));
    HQ_CUDA(cudaMemcpyAsync(ps.range, range.data(), 4 * (G + 1), cudaMemcpyHostToDevice, s));
    HQ_CUDA(cudaMemcpyAsync(&herr, h->d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    cleanup();
    if (herr) {
        ps.release();
        h->err = "rate program overflow (more than 255 groups for a unit)";
        return HQ_I_OVERFLOW;
    }
    ps.cap = hq3_launch::choose_cap(nW, ps.maxblk, h->dev_loop);
    return HQ_OK;
}

static void use_progset(hq_problem *h, ProgSet &ps) {
    dfree(h->d_off16);
    dfree(h->d_range);
    dfree(h->d_prog);
    h->d_off16 = ps.off16;
    h->d_range = ps.range;
    h->d_prog = ps.prog;
    h->total16 = ps.total16;
    h->maxblk_all = ps.maxblk;
    h->maxrec = ps.cap;
    h->prog_nwv = ps.nwv;
    h->prog_bytes = 16.0 * (double)ps.total16;
    ps.off16 = ps.range = nullptr;
    ps.prog = nullptr;
}

// folded scalar step of a path-3 sweep launch (S3Args::fold)
struct FoldArgs {
    int fold = 0;
    int prev_c = 0;
    uint32_t prev_active = 0;
    const double *prev_partial = nullptr;
    double *blk_out = nullptr;
};

static cudaError_t tiled_sweep(hq_problem *h, const S2Args &sa, int mode, cudaStream_t s,
                               const FoldArgs *f = nullptr);
static S2Args base_s2(hq_problem *h);

static hq_status v3_prepare(hq_problem *h, cudaStream_t s) {
    if (h->v2_ready) return HQ_OK;
    const int N = h->N;
    const uint64_t S = 1ull << N;
    const int Nt = N - 9 - h->nW;
    const uint64_t ntiles = 1ull << Nt;
    // CTA tile visit order (DESIGN.md §4 "Tile order").
    //  * popcount order (N < 27): tiles by popcount of the tile index; every CTA takes a
    //    contiguous, work-balanced range of it.  A popcount class of q blocks fits in L2 up to
    //    N = 26, so the tile-unit neighbours of the tiles in flight are L2 hits.
    //  * group order (N >= 27, the default there): "groups" = sub-cubes of the 11 low tile
    //    bits, visited in Gray-code order of the high tile bits; the n-th tile of that sequence
    //    goes to CTA n mod G, so all CTAs work on one group at a time and its q blocks are the
    //    L2 working set (cfg5: 156 -> 110 B/state of DRAM traffic, -8 % per half-sweep).
    //  * chunked order (HQ_ORDER=chunk, the default before the group order): "chunks" =
    //    sub-cubes of the b low tile bits; chunk k goes to CTA k mod G, popcount order of the
    //    low bits inside a chunk.  Each CTA's chunks are contiguous in `order`.
    std::vector<uint32_t> order;
    order.reserve(ntiles);
    auto popcount_order = [](int bits, std::vector<uint32_t> &out) {
        out.push_back(0);
        for (int K = 1; K <= bits; K++) {
            uint64_t x = (1ull << K) - 1;
            while (x < (1ull << bits)) {
                out.push_back((uint32_t)x);
                const uint64_t cc = x & (~x + 1), r = x + cc;
                x = (((r ^ x) >> 2) / cc) | r;
            }
        }
    };
    h->chunk_bits = 0;
    h->chunked = false;
    h->h_in = 32;
    h->h_out_pol = 0;
    h->pf_h = h->pf_o = 0;
    {
        const char *oenv = getenv("HQ_ORDER");
        // default: group order from N = 27 (measured), popcount order below
        const std::string om = oenv ? oenv : (N >= 27 ? "group" : "");
        bool chunked = false;
        if (om == "popcount") chunked = false;
        if (om == "chunk") chunked = true;
        int b = 5;   // measured: cfg4 b = 1 / 3 / 5 -> 2.71 / 2.64 / 2.41 s (popcount order 2.95 s)
        if (const char *benv = getenv("HQ_CHUNK_BITS")) b = atoi(benv);
        b = std::max(0, std::min(b, Nt));
        if (chunked && ((ntiles >> b) < (uint64_t)h->sgrid)) chunked = false;   // too few chunks to spread
        if (om == "group") {
            // groups = sub-cubes of the gb low tile bits, visited in Gray-code order of the
            // high tile bits (consecutive groups are neighbours along one high bit); inside a
            // group the tiles follow the popcount of their low bits.  The n-th tile of this
            // group-major sequence goes to CTA n mod G, so all CTAs work on the same group at
            // the same time: its 2^gb q blocks (and the previous / next group's) are the L2
            // working set, every neighbour along a low tile bit is an L2 hit.
            int gb = 11;
            if (const char *genv = getenv("HQ_GROUP_BITS")) gb = atoi(genv);
            gb = std::max(0, std::min(gb, Nt));
            std::vector<uint32_t> low, seq;
            popcount_order(gb, low);
            const uint64_t ng = ntiles >> gb;
            seq.reserve(ntiles);
            for (uint64_t k = 0; k < ng; k++) {
                const uint64_t gk = k ^ (k >> 1);
                for (uint32_t lo : low) seq.push_back((uint32_t)(gk << gb) | lo);
            }
            const int G = h->sgrid;
            h->chunk_bits = gb;
            h->chunked = true;
            h->h_in = gb;
            h->h_out_pol = 2;
            if (const char *penv = getenv("HQ_HPOL")) h->h_out_pol = atoi(penv);
            h->pf_h = 4;   // measured at cfg5: 4 units ahead -12 % per half-sweep, 6 ahead -9 %
            h->pf_o = 1;
            // group progress bound: CTAs stay within 2 groups of each other (the L2 then holds the
            // live groups: cfg5 -8.6 % per half-sweep, same box; no gain with 16 groups at cfg4)
            h->gs_lag = ng >= 32 ? 2 : 0;
            if (const char *e = getenv("HQ_GLAG")) h->gs_lag = std::max(0, atoi(e));
            h->gs_ng = (uint32_t)ng;
            if (h->sgrid > h->nsm) h->gs_lag = 0;   // the bound needs one resident CTA per SM

            h->chunk_range.assign(G + 1, 0);
            for (int cta = 0; cta < G; cta++) {
                h->chunk_range[cta] = (uint32_t)order.size();
                for (uint64_t n = (uint64_t)cta; n < ntiles; n += (uint64_t)G) order.push_back(seq[n]);
            }
            h->chunk_range[G] = (uint32_t)order.size();
        } else if (om == "natural") {
            // device-resident solve: tiles in natural order, handed out dynamically in units of
            // consecutive tiles, so the CTAs in flight work on neighbouring tiles and the
            // tile-unit neighbours at distance 2^h < L2 window stay L2-resident
            for (uint64_t t = 0; t < ntiles; t++) order.push_back((uint32_t)t);
        } else if (chunked) {
            h->chunk_bits = b;
            h->chunked = true;
            std::vector<uint32_t> low;
            popcount_order(b, low);
            const uint64_t nch = ntiles >> b;
            const int G = h->sgrid;
            h->chunk_range.assign(G + 1, 0);
            for (int cta = 0; cta < G; cta++) {
                h->chunk_range[cta] = (uint32_t)order.size();
                for (uint64_t k = (uint64_t)cta; k < nch; k += (uint64_t)G)
                    for (uint32_t lo : low) order.push_back((uint32_t)(k << b) | lo);
            }
            h->chunk_range[G] = (uint32_t)order.size();
        } else {
            popcount_order(Nt, order);
        }
    }
    if (const char *e = getenv("HQ_PFH")) h->pf_h = atoi(e);
    if (const char *e = getenv("HQ_PFO")) h->pf_o = atoi(e);
    h->in_pol = 0;
    if (const char *e = getenv("HQ_INPOL")) h->in_pol = atoi(e);
    h->pf_min = 0;
    if (const char *e = getenv("HQ_PFMIN")) h->pf_min = atoi(e);
    if (dmalloc((void **)&h->d_order, 4 * ntiles) != cudaSuccess ||
        (!h->full_lists && dmalloc((void **)&h->d_lamarr, 8 * S) != cudaSuccess)) {
        cudaGetLastError();
        h->err = "device memory for the tile tables could not be allocated";
        return HQ_E_NOMEM;
    }
    HQ_CUDA(cudaMemcpyAsync(h->d_order, order.data(), 4 * ntiles, cudaMemcpyHostToDevice, s));
    P2Args pa;
    memset(&pa, 0, sizeof(pa));
    pa.N = N;
    pa.full_lists = h->full_lists ? 1 : 0;
    pa.Lam = h->Lam;
    for (int u = 0; u < 32; u++) pa.nu[u] = u < N ? h->nu_int[u] : 0.0;
    pa.nnodes = (int)h->trie.node.size();
    pa.node = h->d_node;
    pa.lam_thr = h->d_lthr;
    pa.lam_end = h->d_lend;
    cudaEvent_t e0 = h->event(2), e1 = h->event(3);
    HQ_CUDA(cudaEventRecord(e0, s));
    const int g = h->nsm * 8;
    // the scatter weights (and lambda_m) are independent of the rate programs: a side stream
    // builds them while the programs are built and partitioned on s
    if (!h->side) {
        HQ_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
        HQ_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
        HQ_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    }
    HQ_CUDA(cudaEventRecord(h->ev_fork, s));
    HQ_CUDA(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    if (!h->full_lists) HQ_CUDA(hq2_launch::lambda_states(pa, h->d_lamarr, g, h->side));
    HQ_CUDA(hq2_launch::omkap(pa, h->d_lamarr, h->d_omkap, g, h->side));
    HQ_CUDA(cudaEventRecord(h->ev_join, h->side));
    // program granularity: warp programs (warp bits folded; fewer pairs per thread; the
    // default) or CTA programs (warps share one program; HQ_PROG=cta, development A/B).
    const char *env = getenv("HQ_PROG");
    const bool cta_prog = env && std::string(env) == "cta";
    ProgSet a;
    hq_status st = v3_programs(h, s, cta_prog ? h->nW : 0, order, a);
    if (st != HQ_OK) return st;
    if (a.prog) use_progset(h, a);
    if (!hq3_launch::fits_smem(h->nW, h->maxrec, h->dev_loop)) {
        h->err = "tile working set exceeds the shared-memory budget";
        return HQ_E_NUMERIC;
    }
    HQ_CUDA(cudaStreamWaitEvent(s, h->ev_join, 0));
    HQ_CUDA(cudaEventRecord(e1, s));
    HQ_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    h->precompute_ms = ms;
    h->v2_ready = true;
    return HQ_OK;
}

// one sweep / residual launch of the tiled path (hq_v3.cu)
static cudaError_t tiled_sweep(hq_problem *h, const S2Args &sa, int mode, cudaStream_t s, const FoldArgs *f) {
    S3Args a;
    memset(&a, 0, sizeof(a));
    a.N = sa.N;
    a.nW = h->nW;
    a.c = sa.c;
    a.active = sa.active;
    a.ntiles = sa.ntiles;
    a.chunk = 0;
    a.Lam = sa.Lam;
    for (int u = 0; u < 32; u++) a.nu[u] = sa.nu[u];
    a.order = sa.order;
    a.off16 = sa.off16;
    a.prog = sa.prog;
    a.total16 = sa.total16;
    a.maxblk16 = sa.maxrec;
    a.range = h->d_range;
    a.full_lists = sa.full_lists;
    a.warp_programs = (h->prog_nwv == 0) ? 1 : 0;
    a.all_staged = h->maxblk_all <= h->maxrec ? 1 : 0;
    a.h_in = h->h_in;
    a.h_out_pol = h->h_out_pol;
    if (hq3_launch::policies(a.pol) != cudaSuccess) return cudaGetLastError();
    a.pf_h = h->pf_h;
    a.in_pol = h->in_pol;
    a.pf_min = h->pf_min;
    a.pf_o = h->pf_o;
    a.pol_q = a.pol[a.in_pol & 3];
    a.pol_hout = a.pol[a.h_out_pol & 3];
    a.pol_ef = a.pol[2];
    if (h->gs_lag > 0 && h->chunked && h->gs_ng > 0) {
        if (!h->d_gsctr) {
            if (dmalloc((void **)&h->d_gsctr, 8 * (size_t)h->gs_ng) != cudaSuccess ||
                cudaMemset(h->d_gsctr, 0, 8 * (size_t)h->gs_ng) != cudaSuccess) {
                cudaGetLastError();
                dfree(h->d_gsctr);
                h->d_gsctr = nullptr;
                h->gs_lag = 0;   // run without the bound
            }
            h->gs_epoch = 0;
        }
        if (h->d_gsctr) {
            a.gs_ctr = h->d_gsctr;
            a.gs_target = (h->gs_epoch + 1) * (unsigned long long)h->sgrid;
            a.gs_bits = h->chunk_bits;
            a.gs_lag = h->gs_lag;
            a.gs_ng = h->gs_ng;
        }
    }
    if (!h->d_wtime && dmalloc((void **)&h->d_wtime, 8 * 4096) == cudaSuccess) cudaMemset(h->d_wtime, 0, 8 * 4096);
    a.wtime = h->d_wtime;
    a.Q = sa.Q;
    a.P = sa.P;
    a.omkap = sa.omkap;
    a.coef = sa.coef;
    a.partial = sa.partial;
    if (f && f->fold) {
        a.fold = 1;
        a.prev_c = f->prev_c;
        a.prev_active = f->prev_active;
        a.prev_partial = f->prev_partial;
        a.blk_out = f->blk_out;
    }
    const cudaError_t e = hq3_launch::sweep(a, sa.full_lists, mode, h->sgrid, s);
    if (a.gs_ctr) {
        if (e == cudaSuccess) h->gs_epoch++;
        else h->gs_lag = 0;   // a launch that did not run leaves the counters behind: stop using them
    }
    return e;
}

static S2Args base_s2(hq_problem *h) {
    const int N = h->N;
    S2Args sa;
    memset(&sa, 0, sizeof(sa));
    sa.N = N;
    sa.full_lists = h->full_lists ? 1 : 0;
    sa.ntiles = 1ull << (h->path == 3 ? N - 9 - h->nW : N - 8);
    sa.Lam = h->Lam;
    for (int u = 0; u < 32; u++) sa.nu[u] = u < N ? h->nu_int[u] : 0.0;
    sa.order = h->d_order;
    sa.off16 = h->d_off16;
    sa.prog = h->d_prog;
    sa.total16 = h->total16;
    sa.maxrec = h->maxrec;
    sa.coef = h->d_blk;
    sa.partial = h->d_partial;
    return sa;
}

struct SolveOut {
    int sweeps = 0, halfsweeps = 0, launches = 0, nres = 0;
    double updates = 0.0, sweep_ms = 0.0, resid_ms = 0.0, res = INFINITY;
    double kernel_ms = -1.0;   // device loop: the one solve launch (sweep_ms from its phase stamps)
    bool converged = false;
};

static hq_status v2_residual(hq_problem *h, cudaStream_t s, S2Args sa, SolveOut &o) {
    const int N = h->N;
    const uint64_t half = 1ull << (N - 1);
    cudaEvent_t ea = h->event(2 * (size_t)o.halfsweeps), eb = h->event(2 * (size_t)o.halfsweeps + 1);
    HQ_CUDA(cudaEventRecord(ea, s));
    for (int c = 0; c < 2; c++) {
        sa.c = c;
        sa.P = h->d_pw + (c ? half : 0);
        sa.Q = h->d_pw + (c ? 0 : half);
        sa.partial = h->d_partial + (size_t)c * h->sgrid * HQ_NL * HQ_NV;
        HQ_CUDA(tiled_sweep(h, sa, 2, s));
    }
    HQ_CUDA(cudaEventRecord(eb, s));
    HQ_CUDA(hq2_launch::scalars(N, sa.full_lists, h->Lam, 2, 0, 0, 2 * h->sgrid, h->d_partial, h->d_blk, s));
    HQ_CUDA(cudaMemcpyAsync(h->h_blk, h->d_blk, sizeof(double) * V2S_TOTAL, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    float x = 0.f;
    cudaEventElapsedTime(&x, ea, eb);
    o.resid_ms += x;
    o.launches += 3;
    o.nres++;
    o.res = h->h_blk[V2S_MISC + 1];
    return HQ_OK;
}

static hq_status solve_v2(hq_problem *h, double tol, int max_iter, double *pi, cudaStream_t s, SolveOut &o) {
    hq_status st = v3_prepare(h, s);
    if (st != HQ_OK) return st;
    const int N = h->N;
    const uint64_t half = 1ull << (N - 1);
    double *hs = h->h_small;
    // --- init (Algorithm 1 step 2)
    for (int n = 0; n < 32; n++) hs[S_MUSTAR + n] = n <= N ? 1.0 / binom(N, n) : 0.0;
    HQ_CUDA(cudaMemcpyAsync(h->d_small + S_MUSTAR, hs + S_MUSTAR, sizeof(double) * 32, cudaMemcpyHostToDevice, s));
    HQ_CUDA(cudaMemsetAsync(h->d_blk, 0, sizeof(double) * V2S_TOTAL, s));
    KArgs k = base_args(h);
    for (int c = 0; c < 2; c++) {
        class_arrays(h, k, c);
        k.partial = h->d_partial + (size_t)c * h->grid * HQ_NL * HQ_NV;
        k.omkap = h->d_omkap + (c ? half : 0);
        k.lamarr = h->d_lamarr ? h->d_lamarr + (c ? half : 0) : nullptr;
        HQ_CUDA(hqk_launch::init_v2(k, h->grid, s));
    }
    HQ_CUDA(hq2_launch::scalars(N, h->full_lists, h->Lam, 0, 0, 0, 2 * h->grid, h->d_partial, h->d_blk, s));
    o.launches += 3;
    if (getenv("HQ_DEBUG_INIT_ONLY")) {
        HQ_CUDA(cudaStreamSynchronize(s));
        o.res = 1.0;
        return HQ_OK;
    }

    S2Args sa = base_s2(h);

    // path 3 folds the scalar step of half-sweep t into the prologue of launch t + 1
    // (S3Args::fold): the scalar block and the CTA partials are double-buffered; a pending
    // step is resolved by k_scalars2 before the host reads the block or a residual runs.
    // (only where the per-CTA partial reduction is short: <= 48 loads per thread)
    const bool fold = h->path == 3 && !getenv("HQ_NOFOLD") &&
                      (size_t)h->sgrid * (N + 1) * NV2 <= (size_t)48 * (32u << h->nW);
    double *blkp[2] = {h->d_blk, h->d_blk + V2S_TOTAL};
    double *part[2] = {h->d_partial, h->d_partial + (size_t)std::max(h->grid, h->sgrid) * HQ_NL * HQ_NV};
    int cur = 0, pw = 0, pc_prev = 0;
    uint32_t pa_prev = 0;
    bool pending = false;
    auto resolve = [&]() -> cudaError_t {   // complete the pending scalar step into blkp[0]
        if (!pending) return cudaSuccess;
        pending = false;
        const int from = cur;
        cur = 0;
        o.launches++;
        return hq2_launch::scalars(N, h->full_lists ? 1 : 0, h->Lam, 1, pc_prev, pa_prev, h->sgrid, part[pw ^ 1],
                                   blkp[from], s, 1, blkp[0]);
    };

    // convergence checks: the two half-sweeps before a check record |dp|
    int next_check = N + 2 * 12;
    double prev_proxy = -1.0;
    int prev_check = 0, rise = 0;
    for (int t = 1; N >= 2; t++) {
        uint32_t active = 0;
        for (int n = 1; n <= N - 1; n++)
            if (((t - n) & 1) == 0 && n <= t && (t - n) / 2 < max_iter) active |= 1u << n;
        if (!active) break;
        const int c = t & 1;
        sa.c = c;
        sa.active = active;
        sa.P = h->d_pw + (c ? half : 0);
        sa.Q = h->d_pw + (c ? 0 : half);
        sa.omkap = h->d_omkap + (c ? half : 0);
        sa.partial = fold ? part[pw] : h->d_partial;
        sa.coef = fold ? blkp[cur] : h->d_blk;
        FoldArgs fa;
        if (fold && pending) {
            fa.fold = 1;
            fa.prev_c = pc_prev;
            fa.prev_active = pa_prev;
            fa.prev_partial = part[pw ^ 1];
            fa.blk_out = blkp[cur ^ 1];
        }
        const bool checking = tol > 0.0 && t >= next_check - 1;
        HQ_CUDA(cudaEventRecord(h->event(2 * (size_t)o.halfsweeps), s));
        HQ_CUDA(tiled_sweep(h, sa, checking ? 1 : 0, s, &fa));
        HQ_CUDA(cudaEventRecord(h->event(2 * (size_t)o.halfsweeps + 1), s));
        if (fold) {
            if (pending) cur ^= 1;
            pending = true;
            pc_prev = c;
            pa_prev = active;
            pw ^= 1;
        } else {
            HQ_CUDA(hq2_launch::scalars(N, sa.full_lists, h->Lam, 1, c, active, h->sgrid, h->d_partial, h->d_blk, s,
                                        h->path == 3 ? 1 : 0));
            o.launches++;
        }
        o.launches++;
        o.halfsweeps++;
        for (int n = 1; n <= N - 1; n++)
            if ((active >> n) & 1u) o.updates += binom(N, n);
        if ((active >> (N - 1)) & 1u) o.sweeps = (t - (N - 1)) / 2 + 1;
        if (!checking || t < next_check) continue;
        HQ_CUDA(resolve());
        HQ_CUDA(cudaMemcpyAsync(h->h_blk, h->d_blk, sizeof(double) * V2S_TOTAL, cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
        if (h->h_blk[V2S_MISC + 0] != 0.0) {
            h->err = "non-positive or non-finite layer normaliser";
            return HQ_E_NUMERIC;
        }
        const double proxy = h->h_blk[V2S_MISC + 2];
        if (!std::isfinite(proxy)) {
            h->err = "non-finite iterate";
            return HQ_E_NUMERIC;
        }
        double rate = 0.0;   // per half-sweep decay factor
        if (prev_proxy > 0.0 && t > prev_check) rate = std::pow(proxy / prev_proxy, 1.0 / (t - prev_check));
        // divergence guard (Assumption 1, can fail): the proxy grew by > 1.5x
        // at four consecutive checks
        rise = (prev_proxy > 0.0 && proxy > 1.5 * prev_proxy) ? rise + 1 : 0;
        if (rise >= 4) {
            h->err = "the residual proxy grew at four consecutive convergence checks (iteration diverges)";
            return HQ_E_NUMERIC;
        }
        prev_proxy = proxy;
        prev_check = t;
        double level = proxy;
        if (proxy <= 2.0 * tol) {
            sa.coef = h->d_blk;
            st = v2_residual(h, s, sa, o);
            if (st != HQ_OK) return st;
            if (o.res <= tol) {
                o.converged = true;
                break;
            }
            level = o.res;
        }
        int gap = 24;
        if (rate > 0.0 && rate < 0.999) {
            const double need = std::log(tol / level) / std::log(rate);
            gap = std::max(2, (int)std::floor(0.9 * need));
            gap = std::min(gap, 200);
        }
        next_check = t + gap;
    }
    HQ_CUDA(resolve());
    sa.coef = h->d_blk;
    if (!o.converged) {
        st = v2_residual(h, s, sa, o);
        if (st != HQ_OK) return st;
        if (tol > 0.0 && o.res <= tol) o.converged = true;
    }
    // the sticky error flag of the scalar steps (v2_residual copied the block to the host):
    // checked on every exit, not only at scheduled convergence checks
    if (h->h_blk[V2S_MISC + 0] != 0.0) {
        h->err = "non-positive or non-finite layer normaliser";
        return HQ_E_NUMERIC;
    }
    HQ_CUDA(hq2_launch::assemble(N, h->d_pw, h->d_blk + V2S_PN, h->perm.data(), pi, h->nsm * 8, s));
    o.launches++;
    // layer masses for the stats
    for (int n = 0; n <= N; n++) hs[S_PN + n] = h->h_blk[V2S_PN + n + 1];
    return HQ_OK;
}

// ---------------------------------------------------------------------------
// Path 3, device-resident solve: init kernels, then ONE cooperative launch of k_loop3 runs
// every half-sweep, the convergence checks (device-side decision on the fused |dp| proxy) and
// the verification residual; the host synchronises once, at the end.
// ---------------------------------------------------------------------------
static hq_status solve_dev(hq_problem *h, double tol, int max_iter, double *pi, cudaStream_t s, SolveOut &o) {
    hq_status st = v3_prepare(h, s);
    if (st != HQ_OK) return st;
    const int N = h->N;
    const uint64_t half = 1ull << (N - 1);
    const int G = h->sgrid;
    double *hs = h->h_small;
    if (!h->d_ctl) {
        if (dmalloc((void **)&h->d_ctl, sizeof(Ctl3)) != cudaSuccess ||
            dmalloc((void **)&h->d_xg, sizeof(unsigned long long) * HQ_XG_WORDS) != cudaSuccess ||
            pinned_alloc((void **)&h->h_ctl, sizeof(Ctl3)) != cudaSuccess) {
            cudaGetLastError();
            h->err = "device memory for the solve control block could not be allocated";
            return HQ_E_NOMEM;
        }
    }
    // --- init (Algorithm 1 step 2): uniform p, its layer sums, the first scalar step
    for (int n = 0; n < 32; n++) hs[S_MUSTAR + n] = n <= N ? 1.0 / binom(N, n) : 0.0;
    HQ_CUDA(cudaMemcpyAsync(h->d_small + S_MUSTAR, hs + S_MUSTAR, sizeof(double) * 32, cudaMemcpyHostToDevice, s));
    HQ_CUDA(cudaMemsetAsync(h->d_blk, 0, sizeof(double) * V2S_TOTAL, s));
    KArgs k = base_args(h);
    for (int c = 0; c < 2; c++) {
        class_arrays(h, k, c);
        k.partial = h->d_partial + (size_t)c * h->grid * HQ_NL * HQ_NV;
        k.omkap = h->d_omkap + (c ? half : 0);
        k.lamarr = h->d_lamarr ? h->d_lamarr + (c ? half : 0) : nullptr;
        HQ_CUDA(hqk_launch::init_v2(k, h->grid, s));
    }
    HQ_CUDA(hq2_launch::scalars(N, h->full_lists, h->Lam, 0, 0, 0, 2 * h->grid, h->d_partial, h->d_blk, s));
    HQ_CUDA(cudaMemsetAsync(h->d_ctl, 0, sizeof(Ctl3), s));
    HQ_CUDA(cudaMemsetAsync(h->d_xg, 0, sizeof(unsigned long long) * HQ_XG_WORDS, s));
    o.launches += 4;

    S3Args a;
    memset(&a, 0, sizeof(a));
    a.N = N;
    a.nW = h->nW;
    a.ntiles = 1ull << (N - 9 - h->nW);
    a.Lam = h->Lam;
    for (int u = 0; u < 32; u++) a.nu[u] = u < N ? h->nu_int[u] : 0.0;
    a.order = h->d_order;
    a.off16 = h->d_off16;
    a.prog = h->d_prog;
    a.total16 = h->total16;
    a.maxblk16 = h->maxrec;
    a.range = h->d_range;
    a.full_lists = h->full_lists ? 1 : 0;
    a.warp_programs = (h->prog_nwv == 0) ? 1 : 0;
    a.all_staged = h->maxblk_all <= h->maxrec ? 1 : 0;
    a.partial = h->d_partial;
    a.xg = h->d_xg;
    // fixed-point range of the exact sums: every per-layer sum is below M = (Lambda + sum nu)
    // x max(1, (Lambda + sum nu) / min(Lambda, nu_min)) (p <= 1 per layer; omega, kappa <= that
    // ratio; den <= Lambda + sum nu); 2^8 headroom; resolution 2^(xe - 32 HQ_XL)
    {
        double snu = 0.0, numin = INFINITY;
        for (int u = 0; u < N; u++) {
            snu += h->nu_int[u];
            numin = std::min(numin, h->nu_int[u]);
        }
        const double tot = h->Lam + snu;
        const double M = tot * std::max(1.0, tot / std::min(h->Lam, numin));
        a.xe = std::ilogb(M) + 1 + 8;
    }
    a.pw = h->d_pw;
    a.omkap_all = h->d_omkap;
    a.blk = h->d_blk;
    a.ctl = h->d_ctl;
    a.tol = tol;
    a.max_iter = max_iter;
    if (hq3_launch::loop_occupancy(a, a.full_lists) < 1) {
        h->err = "the device-resident solve kernel does not fit an SM";
        return HQ_E_CUDA;
    }
    cudaEvent_t e0 = h->event(0), e1 = h->event(1);
    HQ_CUDA(cudaEventRecord(e0, s));
    HQ_CUDA(hq3_launch::loop(a, a.full_lists, G, s));
    HQ_CUDA(cudaEventRecord(e1, s));
    o.launches += 1;
    HQ_CUDA(cudaMemcpyAsync(h->h_ctl, h->d_ctl, sizeof(Ctl3), cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaMemcpyAsync(h->h_blk, h->d_blk, sizeof(double) * V2S_TOTAL, cudaMemcpyDeviceToHost, s));
    HQ_CUDA(hq2_launch::assemble(N, h->d_pw, h->d_blk + V2S_PN, h->perm.data(), pi, h->nsm * 8, s));
    o.launches += 1;
    HQ_CUDA(cudaStreamSynchronize(s));
    float kms = 0.f;
    cudaEventElapsedTime(&kms, e0, e1);
    const Ctl3 &c = *h->h_ctl;
    o.sweeps = c.sweeps;
    o.halfsweeps = c.halfsweeps;
    o.updates = c.updates;
    o.nres = c.nres;
    o.res = c.res;
    o.converged = c.status == SOLVE3_CONVERGED;
    // time split of the one launch by the globaltimer stamps of CTA 0 (sweep vs residual phases)
    const double tot_ns = (double)c.ns_sweep + (double)c.ns_res;
    o.sweep_ms = tot_ns > 0 ? kms * (double)c.ns_sweep / tot_ns : kms;
    o.resid_ms = tot_ns > 0 ? kms * (double)c.ns_res / tot_ns : 0.0;
    o.kernel_ms = kms;
    for (int n = 0; n <= N; n++) hs[S_PN + n] = h->h_blk[V2S_PN + n + 1];
    if (getenv("HQ_DEBUG_CTL"))
        fprintf(stderr, "k_loop3: status %d sweeps %d halfsweeps %d nres %d phases %d res %.3e proxy %.3e grid %d\n",
                c.status, c.sweeps, c.halfsweeps, c.nres, c.phases, c.res, c.proxy, G);
    if (c.status == SOLVE3_NUMERIC) {
        h->err = c.err ? "non-finite or out-of-range per-layer sum" : "non-positive or non-finite layer normaliser";
        return HQ_E_NUMERIC;
    }
    if (c.status == SOLVE3_NOTDECR) {
        h->err = "the residual proxy grew at four consecutive convergence checks (iteration diverges)";
        return HQ_E_NUMERIC;
    }
    return HQ_OK;
}

// Switch a handle to path 1 (two-pass kernels, per-thread trie walk over the ABI-ordered
// preference trie): used when the tiled paths' rate programs overflow their format
// (more than V3_MAXPAIRS distinct (unit, pattern) pairs in a tile, e.g. thousands of
// unstructured lists).  Slower, but valid for every instance.
static void fallback_path1(hq_problem *h) {
    h->release();
    h->device = -1;
    h->path = 1;
    h->v2 = false;
    h->dev_loop = false;
    h->chunked = false;
    for (int u = 0; u < h->N; u++) h->perm[u] = u;
    h->trie = build_trie(h->N, h->J, h->lam.data(), h->pref.data());
    h->nu_int = h->mu;
}

static hq_status solve_core(hq_handle h, double tol, int max_iter, double *pi, void *cuda_stream, int *iters_out,
                            double *residual_out) {
    if (!h) return HQ_E_INVAL;
    if (!pi) {
        h->err = "pi is NULL";
        return HQ_E_INVAL;
    }
    if (max_iter < 0 || !(tol == tol)) {
        h->err = "max_iter must be >= 0 and tol not NaN";
        return HQ_E_INVAL;
    }
    hq_status st = ensure_device(h);
    if (st != HQ_OK) return st;
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const int N = h->N;
    const size_t S = (size_t)1 << N;
    double *hs = h->h_small;
    if (h->v2) {
        cudaEvent_t a0, a1;
        HQ_CUDA(cudaEventCreate(&a0));
        HQ_CUDA(cudaEventCreate(&a1));
        HQ_CUDA(cudaEventRecord(a0, s));
        SolveOut o;
        st = (h->path == 3 && h->dev_loop) ? solve_dev(h, tol, max_iter, pi, s, o) : solve_v2(h, tol, max_iter, pi, s, o);
        if (st != HQ_OK) {
            cudaEventDestroy(a0);
            cudaEventDestroy(a1);
            if (st == HQ_I_OVERFLOW) {   // rate programs do not fit: the general path for this handle
                fallback_path1(h);
                return solve_core(h, tol, max_iter, pi, cuda_stream, iters_out, residual_out);
            }
            return st;
        }
        HQ_CUDA(cudaEventRecord(a1, s));
        HQ_CUDA(cudaEventSynchronize(a1));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a0, a1);
        cudaEventDestroy(a0);
        cudaEventDestroy(a1);
        double sweep_ms = 0.0;
        if (o.kernel_ms >= 0.0) {
            sweep_ms = o.sweep_ms;
        } else {
            for (int i = 0; i < o.halfsweeps; i++) {
                float x = 0.f;
                cudaEventElapsedTime(&x, h->ev[2 * i], h->ev[2 * i + 1]);
                sweep_ms += x;
            }
        }
        double sp = 0.0;
        for (int n = 0; n <= N; n++) sp += hs[S_PN + n];
        memset(h->stats, 0, sizeof(h->stats));
        h->stats[0] = o.sweeps;
        h->stats[1] = o.halfsweeps;
        h->stats[2] = o.updates;
        h->stats[3] = o.launches;
        h->stats[4] = o.nres;
        h->stats[5] = (double)h->trie.node.size();
        h->stats[6] = sp - 1.0;
        h->stats[7] = ms;
        h->stats[8] = sweep_ms;
        h->stats[9] = o.halfsweeps;
        h->stats[10] = o.resid_ms;
        h->stats[11] = h->precompute_ms;
        h->stats[12] = h->prog_bytes;
        h->stats[13] = h->path;   // path id
        h->stats[14] = h->maxblk_all;
        h->stats[15] = h->prog_nwv;
        h->stats[16] = o.kernel_ms >= 0.0 ? o.kernel_ms : 0.0;
        h->stats[17] = o.kernel_ms >= 0.0 ? 1.0 : 0.0;
        h->stats[18] = h->chunked ? h->chunk_bits : -1;
        h->stats[19] = (h->chunked && h->d_gsctr) ? h->gs_lag : 0;
        if (iters_out) *iters_out = o.sweeps;
        if (residual_out) *residual_out = o.res;
        if (!std::isfinite(o.res)) {
            h->err = "non-finite residual";
            return HQ_E_NUMERIC;
        }
        h->solved = true;
        if (tol <= 0.0) return HQ_OK;
        return o.converged ? HQ_OK : HQ_NOT_CONVERGED;
    }
    cudaEvent_t e0, e1;
    HQ_CUDA(cudaEventCreate(&e0));
    HQ_CUDA(cudaEventCreate(&e1));
    HQ_CUDA(cudaEventRecord(e0, s));
    int launches = 0, nres = 0;
    HQ_CUDA(cudaMemsetAsync(h->d_err, 0, sizeof(int), s));

    // --- init (Algorithm 1 step 2)
    for (int n = 0; n < 32; n++) hs[S_MUSTAR + n] = n <= N ? 1.0 / binom(N, n) : 0.0;
    HQ_CUDA(cudaMemcpyAsync(h->d_small + S_MUSTAR, hs + S_MUSTAR, sizeof(double) * 32, cudaMemcpyHostToDevice, s));
    KArgs k = base_args(h);
    for (int c = 0; c < 2; c++) {
        class_arrays(h, k, c);
        k.partial = h->d_partial + (size_t)c * h->grid * HQ_NL * HQ_NV;
        HQ_CUDA(hqk_launch::init(k, h->grid, s));
        launches++;
    }
    HQ_CUDA(hqk_launch::layer_reduce(N, 0, h->grid, 2, h->d_partial, 2, 2, h->d_small + S_LAM, h->d_small + S_MU,
                                     nullptr, nullptr, h->d_err, s));
    launches++;

    // --- staggered sweeps
    int sweeps = 0, halfsweeps = 0;
    double updates = 0.0;
    double res = INFINITY;
    bool converged = false;
    double dl1_prev = INFINITY;
    int next_check_sweep = 1;
    const double rate_guess = 0.9;
    for (int t = 1; N >= 2; t++) {
        uint32_t active = 0;
        for (int n = 1; n <= N - 1; n++)
            if (((t - n) & 1) == 0 && n <= t && (t - n) / 2 < max_iter) active |= 1u << n;
        if (!active) break;
        const int c = t & 1;
        class_arrays(h, k, c);
        k.active = active;
        k.partial = h->d_partial;
        HQ_CUDA(cudaEventRecord(h->event(2 * (size_t)halfsweeps), s));
        HQ_CUDA(hqk_launch::gather(k, h->grid, s));
        HQ_CUDA(hqk_launch::layer_reduce(N, active, h->grid, 1, h->d_partial, 6, 0, h->d_small + S_LAM,
                                         h->d_small + S_MU, h->d_small + S_MUSTAR, nullptr, h->d_err, s));
        HQ_CUDA(hqk_launch::finalize(k, h->grid, s));
        HQ_CUDA(cudaEventRecord(h->event(2 * (size_t)halfsweeps + 1), s));
        HQ_CUDA(hqk_launch::layer_reduce(N, active, h->grid, 1, h->d_partial, 3, 1, nullptr, nullptr, nullptr,
                                         h->d_small + S_STATS, h->d_err, s));
        launches += 4;
        halfsweeps++;
        for (int n = 1; n <= N - 1; n++)
            if ((active >> n) & 1u) updates += binom(N, n);
        if (!((active >> (N - 1)) & 1u)) continue;
        sweeps = (t - (N - 1)) / 2 + 1;
        if (tol <= 0.0) continue;
        // convergence trigger: L1 change of pi over the last two half-sweeps
        HQ_CUDA(cudaMemcpyAsync(hs, h->d_small, sizeof(double) * S_TOTAL, cudaMemcpyDeviceToHost, s));
        int herr = 0;
        HQ_CUDA(cudaMemcpyAsync(&herr, h->d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
        HQ_CUDA(cudaStreamSynchronize(s));
        if (herr) {
            h->err = "non-positive or non-finite layer normaliser";
            return HQ_E_NUMERIC;
        }
        double pnh[32];
        birth_death(N, hs + S_LAM, hs + S_MU, pnh);
        double dl1 = 0.0;
        for (int n = 1; n <= N - 1; n++) dl1 += pnh[n] * hs[S_STATS + n * 4 + 0];
        if (!std::isfinite(dl1)) {
            h->err = "non-finite iterate";
            return HQ_E_NUMERIC;
        }
        const double proxy = dl1 + dl1_prev;
        dl1_prev = dl1;
        if (sweeps >= next_check_sweep && proxy <= 4.0 * tol) {
            hq_status rs = true_residual(h, s, &res, &launches);
            if (rs != HQ_OK) return rs;
            nres++;
            if (res <= tol) {
                converged = true;
                break;
            }
            // geometric decay: skip ahead by the expected number of sweeps
            const double need = std::log(tol / res) / std::log(rate_guess);
            next_check_sweep = sweeps + std::max(1, (int)std::ceil(need));
        }
    }
    if (!converged) {
        hq_status rs = true_residual(h, s, &res, &launches);
        if (rs != HQ_OK) return rs;
        nres++;
        if (tol > 0.0 && res <= tol) converged = true;
        if (N == 1) converged = true;
    } else {
        // p(n) already on device from the last true residual
    }
    HQ_CUDA(hqk_launch::assemble(N, h->d_pw, h->d_small + S_PN, pi, h->nsm * 8, s));
    launches++;
    HQ_CUDA(cudaEventRecord(e1, s));
    HQ_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    double sweep_ms = 0.0;
    for (int i = 0; i < halfsweeps; i++) {
        float x = 0.f;
        cudaEventElapsedTime(&x, h->ev[2 * i], h->ev[2 * i + 1]);
        sweep_ms += x;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    int herr = 0;
    HQ_CUDA(cudaMemcpy(&herr, h->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (herr) {
        h->err = "non-positive or non-finite layer normaliser";
        return HQ_E_NUMERIC;
    }
    double sp = 0.0;
    for (int n = 0; n <= N; n++) sp += h->h_small[S_PN + n];
    memset(h->stats, 0, sizeof(h->stats));
    h->stats[0] = sweeps;
    h->stats[1] = halfsweeps;
    h->stats[2] = updates;
    h->stats[3] = launches;
    h->stats[4] = nres;
    h->stats[5] = (double)h->trie.node.size();
    h->stats[6] = sp - 1.0;
    h->stats[7] = ms;
    h->stats[8] = sweep_ms;
    h->stats[9] = 2.0 * halfsweeps;   // gather + finalize launches
    h->stats[13] = 1;   // path id
    if (iters_out) *iters_out = sweeps;
    if (residual_out) *residual_out = res;
    if (!std::isfinite(res)) {
        h->err = "non-finite residual";
        return HQ_E_NUMERIC;
    }
    h->solved = true;
    (void)S;
    if (tol <= 0.0) return HQ_OK;
    return converged ? HQ_OK : HQ_NOT_CONVERGED;
}

// Waiting room (Proposition "Reformulation, Finite Buffer", and the
// Remark on unlimited capacity): the conditional probabilities are those of
// the loss system, the tail states follow the birth-death chain with lambda(n) = Lambda and
// mu(n) = sum nu for n > N, so P~{c} = P{all busy} r^c with r = Lambda / sum nu and every
// hypercube probability is the loss-system one scaled by 1 / (1 + sum_c r^c P{all busy}).
static hq_status apply_buffer(hq_problem *h, double *pi, cudaStream_t s) {
    const int N = h->N;
    const uint64_t S = 1ull << N;
    double pN = 0.0;
    HQ_CUDA(cudaMemcpyAsync(&pN, pi + (S - 1), sizeof(double), cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    double snu = 0.0;
    for (int i = 0; i < N; i++) snu += h->mu[i];
    const double r = h->Lam / snu;
    double geo = 0.0;   // sum_{c=1}^{C} r^c (C = infinity: r / (1 - r))
    if (h->bufC < 0) {
        if (!(r < 1.0)) {
            h->err = "unlimited buffer needs Lambda < sum of service rates (PAPER.md:296)";
            return HQ_E_INVAL;
        }
        geo = r / (1.0 - r);
    } else if (h->bufC <= 65536) {
        double x = 1.0;
        for (int c = 1; c <= h->bufC; c++) {
            x *= r;
            geo += x;
        }
    } else {
        geo = r == 1.0 ? (double)h->bufC : r * std::expm1((double)h->bufC * std::log(r)) / (r - 1.0);
    }
    const double sc = 1.0 / (1.0 + pN * geo);
    HQ_CUDA(hqk_launch::scale(pi, S, sc, h->nsm * 8, s));
    h->q_r = r;
    h->q_first = sc * pN * r;
    h->q_mass = sc * pN * geo;
    h->q_last = h->bufC < 0 ? 0.0 : sc * pN * std::pow(r, (double)h->bufC);
    HQ_CUDA(cudaStreamSynchronize(s));
    return HQ_OK;
}

extern "C" hq_status hq_solve(hq_handle h, double tol, int max_iter, double *pi, void *cuda_stream, int *iters_out,
                              double *residual_out) {
    hq_status st = solve_core(h, tol, max_iter, pi, cuda_stream, iters_out, residual_out);
    if (h && h->bufC != 0 && (st == HQ_OK || st == HQ_NOT_CONVERGED)) {
        const hq_status sb = apply_buffer(h, pi, (cudaStream_t)cuda_stream);
        if (sb != HQ_OK) {
            h->solved = false;
            return sb;
        }
    }
    return st;
}

extern "C" hq_status hq_response_times(hq_handle h, const double *dispatch, const double *tau, double T_bar,
                                       double *mrt, double *frac_within, double *mrt_j, double *frac_within_j,
                                       void *cuda_stream) {
    if (!h) return HQ_E_INVAL;
    if (!dispatch || !tau || !mrt || !frac_within || !(T_bar == T_bar)) {
        h->err = "NULL argument or NaN threshold";
        return HQ_E_INVAL;
    }
    if (h->bufC != 0) {
        h->err = "response-time measures are defined for the zero-capacity system (PAPER.md:1015)";
        return HQ_E_INVAL;
    }
    const size_t JN = (size_t)h->J * h->N;
    for (size_t k = 0; k < JN; k++)
        if (!std::isfinite(tau[k]) || tau[k] < 0.0) {
            h->err = "tau must be finite and >= 0";
            return HQ_E_INVAL;
        }
    hq_status st = ensure_device(h);
    if (st != HQ_OK) return st;
    cudaStream_t s = (cudaStream_t)cuda_stream;
    double *d_tau = nullptr, *d_tot = nullptr;
    if (dmalloc((void **)&d_tau, sizeof(double) * JN) != cudaSuccess ||
        dmalloc((void **)&d_tot, sizeof(double) * 2) != cudaSuccess) {
        dfree(d_tau);
        h->err = "device memory for tau could not be allocated";
        return HQ_E_NOMEM;
    }
    double tot[2] = {0.0, 0.0};
    cudaError_t e = cudaMemcpyAsync(d_tau, tau, sizeof(double) * JN, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = hqk_launch::response(h->N, h->J, h->d_lam, h->Lam, dispatch, d_tau, T_bar, mrt_j, frac_within_j, d_tot, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(tot, d_tot, sizeof(tot), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    dfree(d_tau);
    dfree(d_tot);
    if (e != cudaSuccess) {
        h->err = std::string("CUDA error: ") + cudaGetErrorString(e);
        return HQ_E_CUDA;
    }
    *mrt = tot[0];
    *frac_within = tot[1];
    return HQ_OK;
}

extern "C" hq_status hq_set_buffer(hq_handle h, int C) {
    if (!h) return HQ_E_INVAL;
    if (C < HQ_BUFFER_UNLIMITED) {
        h->err = "buffer capacity must be >= 0 or HQ_BUFFER_UNLIMITED";
        return HQ_E_INVAL;
    }
    if (C != 0 && !h->full_lists) {
        h->err = "a waiting room needs full preference lists (a call queues when every unit is busy)";
        return HQ_E_INVAL;
    }
    h->bufC = C;
    h->solved = false;
    return HQ_OK;
}

extern "C" hq_status hq_queue_tail(hq_handle h, double *tail, int len, double *mass) {
    if (!h || len < 0 || (len > 0 && !tail)) return HQ_E_INVAL;
    if (!h->solved) {
        h->err = "hq_queue_tail called before a successful hq_solve";
        return HQ_E_ORDER;
    }
    if (h->bufC > 0 && len > h->bufC) {
        h->err = "len exceeds the buffer capacity";
        return HQ_E_INVAL;
    }
    double x = h->q_first;
    for (int c = 0; c < len; c++) {
        tail[c] = h->bufC == 0 ? 0.0 : x;
        x *= h->q_r;
    }
    if (mass) *mass = h->bufC == 0 ? 0.0 : h->q_mass;
    return HQ_OK;
}

extern "C" hq_status hq_measures(hq_handle h, const double *pi, double *workload, double *dispatch, double *loss,
                                 void *cuda_stream) {
    if (!h) return HQ_E_INVAL;
    if (!h->solved) {
        h->err = "hq_measures called before a successful hq_solve";
        return HQ_E_ORDER;
    }
    if (!pi || !workload || !dispatch || !loss) {
        h->err = "NULL argument";
        return HQ_E_INVAL;
    }
    hq_status st = ensure_device(h);
    if (st != HQ_OK) return st;
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const int N = h->N;
    const size_t S = (size_t)1 << N;
    double *g = h->d_pw;   // p is re-initialised by every hq_solve, so it can hold the superset sums
    HQ_CUDA(cudaMemcpyAsync(g, pi, sizeof(double) * S, cudaMemcpyDeviceToDevice, s));
    HQ_CUDA(hqk_launch::zeta(N, g, h->nsm * 8, s));
    HQ_CUDA(hqk_launch::measures(N, h->J, h->d_lam, h->Lam, h->d_pref, g, workload, dispatch,
                                 h->d_small + S_STATS, s));
    if (h->bufC != 0) {   // waiting room: queued calls (R14), loss = P~{C}
        HQ_CUDA(hqk_launch::buffer_measures(N, h->J, h->d_lam, h->Lam, h->mu.data(), pi + (S - 1), h->d_small + S_STATS,
                                            h->q_mass, h->q_last, h->q_last, workload, dispatch, s));
        HQ_CUDA(cudaStreamSynchronize(s));
        *loss = h->q_last;
        return HQ_OK;
    }
    HQ_CUDA(cudaMemcpyAsync(loss, h->d_small + S_STATS, sizeof(double), cudaMemcpyDeviceToHost, s));
    HQ_CUDA(cudaStreamSynchronize(s));
    return HQ_OK;
}

extern "C" void hq_destroy(hq_handle h) { delete h; }

extern "C" const char *hq_error_string(hq_handle h) {
    if (!h) return g_create_error.c_str();
    return h->err.c_str();
}

extern "C" hq_status hq_stats(hq_handle h, double *out) {
    if (!h || !out) return HQ_E_INVAL;
    memcpy(out, h->stats, sizeof(h->stats));
    return HQ_OK;
}

// Debug/introspection copy of internal device arrays (tests only).
//   which: 0 v2 scalar block, 1 p (parity-compressed), 2 (omega, kappa),
//          3 rate programs, 4 program offsets, 5 tile order, 6 internal->ABI unit map (host)
extern "C" hq_status hq_debug_copy(hq_handle h, int which, void *host, size_t bytes) {
    if (!h || !host) return HQ_E_INVAL;
    const void *src = nullptr;
    if (which == 6) {
        memcpy(host, h->perm.data(), std::min(bytes, sizeof(int) * h->perm.size()));
        return HQ_OK;
    }
    switch (which) {
        case 0: src = h->d_blk; break;
        case 1: src = h->d_pw; break;
        case 2: src = h->d_omkap; break;
        case 3: src = h->d_prog; break;
        case 4: src = h->d_off16; break;
        case 5: src = h->d_order; break;
        case 7: src = h->d_wtime; break;
        case 8: src = h->d_range; break;
        default: return HQ_E_INVAL;
    }
    if (!src) return HQ_E_ORDER;
    cudaError_t e = cudaMemcpy(host, src, bytes, cudaMemcpyDeviceToHost);
    return e == cudaSuccess ? HQ_OK : HQ_E_CUDA;
}

extern "C" const char *hq_version(void) { return "hq-b200 0.1 (sm_100a, fp64, red-black staggered Algorithm 1)"; }
