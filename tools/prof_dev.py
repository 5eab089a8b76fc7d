"""Profiling driver for the device-resident solve: one hq_solve of a BASELINE config for a
fixed number of sweeps (tol = 0).  python tools/prof_dev.py CFG SWEEPS"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hqinst  # noqa: E402
from paper_2603_03019_b200 import hq  # noqa: E402

cfg = int(sys.argv[1])
sweeps = int(sys.argv[2])
inst = hqinst.config_instance(cfg)
s = hq.Solver.from_instance(inst)
pi = torch.empty(1 << inst.N, dtype=torch.float64, device="cuda")
r = s.solve(tol=0.0, max_iter=sweeps, pi=pi)
torch.cuda.synchronize()
print(json.dumps(dict(cfg=cfg, iters=r["iters"], residual=r["residual"], stats=s.stats())))
s.close()
