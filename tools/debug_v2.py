"""Debug aid for the tiled (v2) path: compares internal device arrays against
straightforward numpy/oracle evaluations on a small instance.  Not a test."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import hqinst, oracle
from paper_2603_03019_b200 import hq

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10
L = int(sys.argv[2]) if len(sys.argv) > 2 else 0
inst = hqinst.generate(N, 25, seed=5, rho=0.6, L=(L or None))
S = 1 << N; half = S >> 1
s = hq.Solver.from_instance(inst)
pi = torch.empty(S, dtype=torch.float64, device="cuda")
os.environ["HQ_DEBUG_INIT_ONLY"] = "1" if len(sys.argv) > 3 else ""
if not os.environ["HQ_DEBUG_INIT_ONLY"]:
    del os.environ["HQ_DEBUG_INIT_ONLY"]
try:
    r = s.solve(tol=0.0, max_iter=0, pi=pi)
    print("solve(max_iter=0):", r["status"], r["residual"])
except Exception as e:
    print("solve failed:", e)
perm = hq.hq_debug_copy(s.h, 6, 4 * N, np.int32)
print("perm", perm)
blk = hq.hq_debug_copy(s.h, 0, 8 * 416, np.float64)
names = dict(LAM=0, MU=32, ALPHA=64, BETA=96, PN=128, OM=176, KA=208, DL1=240, SUMP=272, MUSTAR=368)
for k, o in names.items():
    print(k, np.round(blk[o:o + N + 2], 6))
print("MISC", blk[400:404])

# internal-order instance
inv = np.zeros(N, int); inv[perm] = np.arange(N)
nu_i = inst.mu[perm]
def m_abi(m):
    return sum(((m >> u) & 1) << perm[u] for u in range(N))
# omega/kappa reference
W = {}
lam_s = np.zeros(S); mu_s = np.zeros(S)
for m in range(S):
    ma = m_abi(m)
    out, lost = oracle.out_rates(inst, ma)
    lam_s[m] = out.sum()
    mu_s[m] = sum(nu_i[u] for u in range(N) if (m >> u) & 1)
den = lam_s + mu_s
om = np.zeros(S); ka = np.zeros(S)
for l in range(S):
    out, _ = oracle.out_rates(inst, m_abi(l))
    for u in range(N):
        if (l >> u) & 1:
            ka[l] += nu_i[u] / den[l ^ (1 << u)]
        else:
            om[l] += out[perm[u]] / den[l | (1 << u)]
ok = hq.hq_debug_copy(s.h, 2, 16 * S, np.float64).reshape(S, 2)
# device layout [class][j], state m: class = popcount parity, j = m >> 1
dev_om = np.zeros(S); dev_ka = np.zeros(S)
for m in range(S):
    c = bin(m).count("1") & 1
    x = (half if c else 0) + (m >> 1)
    dev_om[m], dev_ka[m] = ok[x]
print("omega max err", np.abs(dev_om - om).max(), "kappa max err", np.abs(dev_ka - ka).max())

# programs: evaluate W_u(m) from the program for every state and compare with Algorithm 3
order = hq.hq_debug_copy(s.h, 5, 4 * (1 << (N - 8)), np.uint32)
off = hq.hq_debug_copy(s.h, 4, 4 * (1 << (N - 8)), np.uint32)
nt = 1 << (N - 8)
total16 = int(s.stats()["program_bytes"]) // 16
prog = hq.hq_debug_copy(s.h, 3, 16 * total16, np.uint32).reshape(-1, 4)
maxerr = 0.0
for i in range(nt):
    t = int(order[i]); o = int(off[i])
    cw = prog[o:o + 8].reshape(-1)
    cnt = [(int(cw[u]) & 0xffff) + (int(cw[u]) >> 16) for u in range(32)]
    cls = [(int(cw[u]) & 0xffff) for u in range(32)]
    w0 = prog[o + 8:o + 24].reshape(-1).view(np.float64)
    pp = o + 24
    pairs = {}
    for u in range(N + 1):
        pairs[u] = []
        for k in range(cnt[u]):
            rec = prog[pp + k]
            c = np.array([rec[0], rec[1]], dtype=np.uint32).view(np.float64)[0]
            pairs[u].append((c, int(rec[2]), k < cls[u]))
        pp += cnt[u]
    for cls in (0, 1):
        for r in range(4):
            for lane in range(32):
                j = (t << 7) | (r << 5) | lane
                b0 = cls ^ (bin(j).count("1") & 1)
                m = (j << 1) | b0
                beta = (cls ^ bin(t).count("1") ^ bin(lane).count("1")) & 1
                Wref = oracle.dispatch_rates(inst, m_abi(m))
                for u in range(N):
                    if not (m >> u) & 1:
                        continue
                    w = w0[u]
                    for c, wd, laneonly in pairs[u]:
                        tl = ((wd & 31) & ~lane) == 0
                        if laneonly:
                            if tl:
                                w += c
                            continue
                        m4 = ((wd >> (8 + 4 * beta)) & 15) if tl else 0
                        if (m4 >> r) & 1:
                            w += c
                    e = abs(w - Wref[perm[u]])
                    if e > 1e-12 and maxerr <= 1e-12:
                        print("first W mismatch: tile", t, "cls", cls, "r", r, "lane", lane, "u", u, "m", bin(m),
                              "W", w, "ref", Wref[perm[u]], "W0", w0[u], "pairs", pairs[u][:6], "cnt", cnt[:N+1])
                    maxerr = max(maxerr, e)
print("program W max err", maxerr)
