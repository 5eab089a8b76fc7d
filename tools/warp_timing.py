"""Per-warp busy cycles of the sweep kernel (library built with -DHQ_WARP_TIMING):
python tools/warp_timing.py CFG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hqinst  # noqa: E402
from paper_2603_03019_b200 import hq  # noqa: E402

inst = hqinst.config_instance(int(sys.argv[1]))
s = hq.Solver.from_instance(inst)
pi = torch.empty(1 << inst.N, dtype=torch.float64, device="cuda")
s.solve(tol=1e-13, max_iter=5000, pi=pi)
w = hq.hq_debug_copy(s.h, 7, 8 * 148 * 16, np.uint64).reshape(148, 16).astype(float)
w = w[w.sum(axis=1) > 0]
print("per-warp-index mean (relative):", np.round(w.mean(axis=0) / w.mean(), 3))
print("CTA max/mean warp:", np.round((w.max(axis=1) / w.mean(axis=1)).mean(), 3),
      " CTA totals max/mean:", np.round(w.sum(axis=1).max() / w.sum(axis=1).mean(), 3))

# per-CTA measured busy cycles against the host's per-tile cost model
G = 148
rng_ = hq.hq_debug_copy(s.h, 8, 4 * (G + 1), np.uint32).astype(np.int64)
st = hq.hq_stats(s.h)
nW = 4
ntiles = 1 << (inst.N - 9 - nW)
off = hq.hq_debug_copy(s.h, 4, 4 * (ntiles << nW), np.uint32).astype(np.int64)
tot16 = int(st[12] // 16)
sz = np.diff(np.append(off, tot16)).reshape(ntiles, 1 << nW)
cost = 380 + sz.max(axis=1)
pred = np.array([cost[rng_[b]:rng_[b + 1]].sum() for b in range(G)])
meas = hq.hq_debug_copy(s.h, 7, 8 * 148 * 16, np.uint64).reshape(148, 16).astype(float).sum(axis=1)
ntl = np.diff(rng_)
print("tiles per CTA min/max:", ntl.min(), ntl.max())
print("pred max/mean:", round(pred.max() / pred.mean(), 3), " corr(pred, meas):", round(np.corrcoef(pred, meas)[0, 1], 3))
order = np.argsort(meas)[::-1][:6]
print("slowest CTAs (meas/mean, pred/mean, tiles, first tile index):",
      [(int(b), round(meas[b] / meas.mean(), 2), round(pred[b] / pred.mean(), 2), int(ntl[b]), int(rng_[b])) for b in order])
# measured cost per tile popcount class
bsum = np.array([sz.max(axis=1)[rng_[b]:rng_[b + 1]].sum() for b in range(G)])
Xm = np.stack([ntl.astype(float), bsum.astype(float)], axis=1)
coef, *_ = np.linalg.lstsq(Xm, meas, rcond=None)
print("fit: cycles = %.0f per tile + %.1f per max-warp record  -> base = %.0f records" % (coef[0], coef[1], coef[0] / coef[1]))
fit = Xm @ coef
print("fit corr:", round(np.corrcoef(fit, meas)[0, 1], 3))

# CTA start / end times of the last MODE-0 launch (globaltimer, ns)
se = hq.hq_debug_copy(s.h, 7, 8 * 4096, np.uint64)[2368:2368 + 2 * G].reshape(G, 2).astype(np.int64)
t0 = se[:, 0].min()
dur = se[:, 1] - se[:, 0]
print("CTA start spread us:", (se[:, 0].max() - t0) / 1e3, " durations us mean/max:", dur.mean() / 1e3, dur.max() / 1e3,
      " last end us:", (se[:, 1].max() - t0) / 1e3)
print("CTA end times (us, sorted, every 10th):", np.round(np.sort(se[:, 1] - t0)[::10] / 1e3, 1))
