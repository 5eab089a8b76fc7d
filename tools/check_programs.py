"""Validate the CTA-tile rate programs (hq_v3.h table format) produced on the GPU against
Algorithm 3 rates from the oracle, for every state of sampled tiles.
Development aid: python tools/check_programs.py N J [L] [ntiles]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["HQ_DEBUG_INIT_ONLY"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hqinst  # noqa: E402
import oracle  # noqa: E402
from paper_2603_03019_b200 import hq  # noqa: E402


def pext(x, M):
    r, j = 0, 0
    for b in range(9):
        if (M >> b) & 1:
            r |= ((x >> b) & 1) << j
            j += 1
    return r


N = int(sys.argv[1]); J = int(sys.argv[2]); L = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "0" else None
nsamp = int(sys.argv[4]) if len(sys.argv) > 4 else 4
inst = hqinst.generate(N, J, seed=11, rho=0.6, L=L)
s = hq.Solver.from_instance(inst)
pi = torch.empty(1 << N, dtype=torch.float64, device="cuda")
s.solve(tol=0.0, max_iter=1, pi=pi)
st = hq.hq_stats(s.h)
nW = max(0, min(4, N - 17, N - 9))
T = 8 + nW
nt = 1 << (N - 1 - T)
perm = hq.hq_debug_copy(s.h, 6, 4 * N, np.int32)
order = hq.hq_debug_copy(s.h, 5, 4 * nt, np.uint32)
off = hq.hq_debug_copy(s.h, 4, 4 * nt, np.uint32)
total16 = int(st[12] // 16)
prog = hq.hq_debug_copy(s.h, 3, 16 * total16, np.uint32).reshape(-1, 4)
print("N", N, "nW", nW, "tiles", nt, "prog records", total16, "perm", perm)
rng = np.random.default_rng(0)
bad = 0
for i in rng.choice(nt, size=min(nsamp, nt), replace=False):
    t = int(order[i]); o = int(off[i])
    info = prog[o:o + 8].reshape(-1)
    infm = prog[o + 25:o + 33].reshape(-1)
    W0 = prog[o + 8:o + 24].copy().view(np.float64).reshape(-1)
    for w in range(1 << nW):
        for lane in range(32):
            tb = lane | (w << 5)
            for r in range(8):
                for c in (0, 1):
                    j = (t << T) | (w << 8) | ((r >> 1) << 6) | (lane << 1) | (r & 1)
                    b0 = c ^ (bin(j).count("1") & 1)
                    m = (j << 1) | b0
                    beta = c ^ ((bin(t).count("1") + bin(lane).count("1") + bin(w).count("1")) & 1)
                    ma = 0
                    for u in range(N):
                        if (m >> u) & 1:
                            ma |= 1 << int(perm[u])
                    Wref = oracle.dispatch_rates(inst, ma)
                    for u in range(N):
                        if not (m >> u) & 1:
                            continue
                        inf = int(info[u])
                        wv = W0[u]
                        if 2 <= u <= 6 and not (lane >> (u - 2)) & 1:
                            wv = 0.0
                        if inf:
                            d = o + 33 + ((inf >> 8) & 0xffff)
                            if inf >> 31:
                                M = int(infm[u])
                                wv = prog[d:d + 64].copy().view(np.float64).reshape(-1)[pext(tb, M)]
                                d += ((1 << bin(M).count("1")) + 1) >> 1
                            for g in range(inf & 0xff):
                                hd = int(prog[d][0]); rm = hd & 0xffff; M = (hd >> 16) & 0x1ff
                                tab = prog[d + 1:d + 1 + 256].copy().view(np.float64).reshape(-1)
                                if (rm >> (8 * beta + r)) & 1:
                                    wv += tab[pext(tb, M)]
                                d += 1 + (((1 << bin(M).count("1")) + 1) >> 1)
                        ref = Wref[int(perm[u])]
                        if abs(wv - ref) > 1e-12 * max(1.0, abs(ref)):
                            bad += 1
                            if bad < 10:
                                print("mismatch tile", t, "warp", w, "lane", lane, "r", r, "c", c, "unit", u, wv, ref)
print("bad", bad)
