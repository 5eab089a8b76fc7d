"""Validate the per-warp-tile rate programs (hq_v3.h table format) produced on the
GPU against Algorithm 3 rates from the oracle, for every state of sampled warp tiles.
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

N = int(sys.argv[1]); J = int(sys.argv[2]); L = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "0" else None
nsamp = int(sys.argv[4]) if len(sys.argv) > 4 else 8
inst = hqinst.generate(N, J, seed=11, rho=0.6, L=L)
s = hq.Solver.from_instance(inst)
pi = torch.empty(1 << N, dtype=torch.float64, device="cuda")
s.solve(tol=0.0, max_iter=1, pi=pi)
st = hq.hq_stats(s.h)
nprog = 1 << (N - 9)
perm = hq.hq_debug_copy(s.h, 6, 4 * N, np.int32)
order = hq.hq_debug_copy(s.h, 5, 4 * nprog, np.uint32)
off = hq.hq_debug_copy(s.h, 4, 4 * nprog, np.uint32)
total16 = int(st[12] // 16)
prog = hq.hq_debug_copy(s.h, 3, 16 * total16, np.uint32).reshape(-1, 4)
print("N", N, "prog records", total16, "perm", perm)
rng = np.random.default_rng(0)
bad = 0
for i in rng.choice(nprog, size=min(nsamp, nprog), replace=False):
    tp = int(order[i])
    o = int(off[i])
    hdr = prog[o:o + 25]
    info = hdr[0:8].reshape(-1)
    W0 = hdr[8:24].copy().view(np.float64).reshape(-1)
    for lane in range(32):
        for r in range(8):
            for c in (0, 1):
                j = (tp << 8) | ((r >> 1) << 6) | (lane << 1) | (r & 1)
                b0 = c ^ (bin(j).count("1") & 1)
                m = (j << 1) | b0
                beta = c ^ ((bin(tp).count("1") + bin(lane).count("1")) & 1)
                ma = 0
                for u in range(N):
                    if (m >> u) & 1:
                        ma |= 1 << int(perm[u])
                Wref = oracle.dispatch_rates(inst, ma)
                for u in range(N):
                    if not (m >> u) & 1:
                        continue
                    inf = int(info[u])
                    w = 0.0 if (2 <= u <= 6 and not (lane >> (u - 2)) & 1) else W0[u]
                    if inf:
                        d = o + 25 + ((inf >> 8) & 0xffff)
                        if inf >> 31:
                            w = prog[d:d + 16].copy().view(np.float64).reshape(-1)[lane]
                            d += 16
                        for g in range(inf & 0xff):
                            rm = int(prog[d][0])
                            tab = prog[d + 1:d + 17].copy().view(np.float64).reshape(-1)
                            if (rm >> (8 * beta + r)) & 1:
                                w += tab[lane]
                            d += 17
                    ref = Wref[int(perm[u])]
                    if abs(w - ref) > 1e-12 * max(1.0, abs(ref)):
                        bad += 1
                        if bad < 10:
                            print("mismatch tile", tp, "lane", lane, "r", r, "c", c, "unit", u, w, ref)
print("bad", bad)
