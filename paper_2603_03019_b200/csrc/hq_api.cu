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
int tile_states();
}  // namespace hqk_launch

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
    out.node.resize(nn);
    out.lam_thr.resize(nn);
    out.lam_end.resize(nn);
    for (int p = 0; p < nn; p++) {
        const int v = order[p];
        out.node[p] = make_int2(t[v].unit, p + size[v]);
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

}  // namespace

struct hq_problem {
    int N = 0, J = 0;
    double Lam = 0.0;
    bool full_lists = true;
    std::vector<double> lam, mu;
    std::vector<int32_t> pref;
    TrieHost trie;
    std::string err;
    int device = -1;
    int nsm = 0;
    bool solved = false;
    double stats[HQ_STATS_LEN] = {0};
    // device memory
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

    ~hq_problem() { release(); }
    void release() {
        cudaFree(d_node);
        cudaFree(d_lthr);
        cudaFree(d_lend);
        cudaFree(d_lam);
        cudaFree(d_pref);
        cudaFree(d_pw);
        cudaFree(d_ab);
        cudaFree(d_partial);
        cudaFree(d_small);
        cudaFree(d_err);
        if (h_small) cudaFreeHost(h_small);
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
enum { S_LAM = 0, S_MU = 32, S_MUSTAR = 64, S_PN = 96, S_STATS = 128, S_INVC = 256, S_TOTAL = 288 };

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
    h->trie = build_trie(N, J, lambda, pref);
    *out = h.release();
    return HQ_OK;
}

static hq_status ensure_device(hq_problem *h) {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        h->err = std::string("no CUDA device: ") + cudaGetErrorString(e);
        return HQ_E_CUDA;
    }
    if (h->device == dev && h->d_pw) return HQ_OK;
    if (h->device != -1 && h->device != dev) h->release();
    h->device = dev;
    HQ_CUDA(cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, dev));
    const int N = h->N;
    const size_t S = (size_t)1 << N;
    const uint64_t ntiles = ((S >> 1) + hqk_launch::tile_states() - 1) / hqk_launch::tile_states();
    h->grid = (int)std::min<uint64_t>(ntiles, (uint64_t)h->nsm * 4);
    const size_t nn = h->trie.node.size();
    auto alloc = [&](void **p, size_t bytes) -> cudaError_t { return cudaMalloc(p, bytes ? bytes : 16); };
    if (alloc((void **)&h->d_pw, sizeof(double) * S) != cudaSuccess ||
        alloc((void **)&h->d_ab, sizeof(double2) * (S >> 1 ? S >> 1 : 1)) != cudaSuccess) {
        cudaGetLastError();
        h->release();
        h->device = -1;
        h->err = "device memory for the working set (2^N doubles x 2) could not be allocated";
        return HQ_E_NOMEM;
    }
    HQ_CUDA(alloc((void **)&h->d_node, sizeof(int2) * nn));
    HQ_CUDA(alloc((void **)&h->d_lthr, sizeof(double) * nn));
    HQ_CUDA(alloc((void **)&h->d_lend, sizeof(double) * nn));
    HQ_CUDA(alloc((void **)&h->d_lam, sizeof(double) * h->J));
    HQ_CUDA(alloc((void **)&h->d_pref, sizeof(int32_t) * h->J * N));
    HQ_CUDA(alloc((void **)&h->d_partial, sizeof(double) * 2 * h->grid * HQ_NL * HQ_NV));
    HQ_CUDA(alloc((void **)&h->d_small, sizeof(double) * S_TOTAL));
    HQ_CUDA(alloc((void **)&h->d_err, sizeof(int)));
    HQ_CUDA(cudaMallocHost((void **)&h->h_small, sizeof(double) * S_TOTAL));
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
    for (int i = 0; i < 32; i++) k.nu[i] = i < h->N ? h->mu[i] : 0.0;
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

extern "C" hq_status hq_solve(hq_handle h, double tol, int max_iter, double *pi, void *cuda_stream, int *iters_out,
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
        HQ_CUDA(hqk_launch::gather(k, h->grid, s));
        HQ_CUDA(hqk_launch::layer_reduce(N, active, h->grid, 1, h->d_partial, 6, 0, h->d_small + S_LAM,
                                         h->d_small + S_MU, h->d_small + S_MUSTAR, nullptr, h->d_err, s));
        HQ_CUDA(hqk_launch::finalize(k, h->grid, s));
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
    double *g = reinterpret_cast<double *>(h->d_ab);   // 2^(N-1) double2 == 2^N doubles
    HQ_CUDA(cudaMemcpyAsync(g, pi, sizeof(double) * S, cudaMemcpyDeviceToDevice, s));
    HQ_CUDA(hqk_launch::zeta(N, g, h->nsm * 8, s));
    HQ_CUDA(hqk_launch::measures(N, h->J, h->d_lam, h->Lam, h->d_pref, g, workload, dispatch,
                                 h->d_small + S_STATS, s));
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

extern "C" const char *hq_version(void) { return "hq-b200 0.1 (sm_100a, fp64, red-black staggered Algorithm 1)"; }
