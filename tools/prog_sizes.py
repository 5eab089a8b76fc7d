"""Distribution of per-CTA-tile program block sizes (records) against the staged capacity:
python tools/prog_sizes.py CFG.  Development aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import hqinst  # noqa: E402
from paper_2603_03019_b200 import hq  # noqa: E402

cfg = int(sys.argv[1])
inst = hqinst.config_instance(cfg)
s = hq.Solver.from_instance(inst)
s.solve(tol=0.0, max_iter=1)
st = hq.hq_stats(s.h)
nW = 4 if inst.N >= 21 else max(0, inst.N - 17)
ntiles = 1 << (inst.N - 9 - nW)
off = hq.hq_debug_copy(s.h, 4, 4 * (ntiles << nW), np.uint32).astype(np.int64)
tot16 = int(st[12] // 16)
starts = off[:: 1 << nW]
blk = np.diff(np.append(starts, tot16))
print("tiles", ntiles, "records total", tot16, "max block", blk.max(), "mean", blk.mean())
for q in [50, 75, 90, 95, 99]:
    print(f"p{q}", np.percentile(blk, q))
for cap in [1024, 2048, 2688, 4096, 6000]:
    over = blk > cap
    print(f"cap {cap}: tiles over {over.mean():.3f}, records in them {blk[over].sum() / blk.sum():.3f}")
