"""Per-warp-index average rate-program size (records) of a config: a proxy of the
per-warp work imbalance inside a CTA tile.  python tools/warp_balance.py CFG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["HQ_DEBUG_INIT_ONLY"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hqinst  # noqa: E402
from paper_2603_03019_b200 import hq  # noqa: E402

inst = hqinst.config_instance(int(sys.argv[1]))
s = hq.Solver.from_instance(inst)
pi = torch.empty(1 << inst.N, dtype=torch.float64, device="cuda")
s.solve(tol=0.0, max_iter=1, pi=pi)
nprog = 1 << (inst.N - 9)
st = hq.hq_stats(s.h)
off = hq.hq_debug_copy(s.h, 4, 4 * nprog, np.uint32).astype(np.int64)
tot = int(st[12] // 16)
size = np.diff(np.append(off, tot))
W = 16
per = size.reshape(-1, W)
print("mean records per warp index:", np.round(per.mean(axis=0), 1))
print("max/mean over warps of the per-tile max:", (per.max(axis=1) / per.mean(axis=1)).mean())
