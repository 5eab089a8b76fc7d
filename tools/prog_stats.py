"""Statistics of the per-warp-tile rate programs (hq_v3.h format) of a BASELINE config:
python tools/prog_stats.py CFG.  Development aid (GPU box).

Per (program, unit): uniform (no data), lane table (|M| bits), register-dependent groups
(count, |M_g|); weighted by the number of warp tiles."""
import collections
import json
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
N = inst.N
nW = 4 if N >= 21 else max(0, N - 17)
ntiles = 1 << (N - 9 - nW)
nprog = ntiles << nW
off = hq.hq_debug_copy(s.h, 4, 4 * nprog, np.uint32).astype(np.int64)
tot16 = int(st[12] // 16)
prog = hq.hq_debug_copy(s.h, 3, 16 * tot16, np.uint32).reshape(-1, 4)
order = hq.hq_debug_copy(s.h, 5, 4 * ntiles, np.uint32)
rng = np.random.default_rng(0)
sample = rng.choice(nprog, size=min(nprog, 4000), replace=False)
c = collections.Counter()
mt = collections.Counter()
mg = collections.Counter()
ngs = collections.Counter()
busy_units = 0
for p in sample:
    o = int(off[p])
    t = int(order[p >> nW])
    for u in range(N + (0 if inst.pref.min() >= 0 else 1)):
        info, M = int(prog[o + u, 0]), int(prog[o + u, 1])
        c["unit-programs"] += 1
        if info == 0:
            c["uniform"] += 1
            continue
        start, ng, tab = (info >> 8) & 0xFFFF, info & 0xFF, info >> 31
        d = o + 33 + start
        if tab:
            c["table"] += 1
            mt[bin(M).count("1")] += 1
            d += ((1 << bin(M).count("1")) + 1) >> 1
        ngs[ng] += 1
        for g in range(ng):
            hd = int(prog[d, 0])
            Mg = (hd >> 16) & 0x1FF
            mg[bin(Mg).count("1")] += 1
            d += 1 + (((1 << bin(Mg).count("1")) + 1) >> 1)
        if ng:
            c["with-groups"] += 1
blocks = np.diff(np.append(off[:: 1 << nW], tot16))
print(json.dumps(dict(cfg=cfg, N=N, programs=int(nprog), records=tot16, mean_block=float(blocks.mean()),
                      counts=dict(c), table_bits=dict(sorted(mt.items())), group_bits=dict(sorted(mg.items())),
                      groups_per_unit=dict(sorted(ngs.items())),
                      groups_per_program=sum(k * v for k, v in ngs.items()) / len(sample))))
