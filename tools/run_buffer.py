"""Cost of the waiting-room post-processing at a BASELINE config: solve with C = 0,
C = 20 and unlimited; prints solve times (CUDA events inside hq_solve) and the
measured extra time.  python tools/run_buffer.py CFG.  Development aid."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hqinst  # noqa: E402
from paper_2603_03019_b200 import hq  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
inst = hqinst.config_instance(cfg)
s = hq.Solver.from_instance(inst)
pi = torch.empty(1 << inst.N, dtype=torch.float64, device="cuda")
out = {}
for C in [0, 20, hq.HQ_BUFFER_UNLIMITED, 0]:
    s.set_buffer(C)
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = s.solve(tol=1e-13, max_iter=5000, pi=pi)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    tail, mass = s.queue_tail(5 if C != 0 else 0)
    out[str(C)] = dict(wall_ms=min(ts), solve_ms_events=s.stats()["solve_ms"], iters=r["iters"],
                       residual=r["residual"], tail_mass=mass, tail=list(tail))
print(json.dumps(dict(cfg=cfg, runs=out), indent=1))
