"""Solve one BASELINE config to tol on cuda:0 and print stats (development aid)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hqinst  # noqa: E402
from paper_2603_03019_b200 import hq  # noqa: E402

cfg = int(sys.argv[1])
rho = float(sys.argv[2]) if len(sys.argv) > 2 else None
inst = hqinst.config_instance(cfg, rho=rho)
t0 = time.time()
s = hq.Solver.from_instance(inst)
pi = torch.empty(1 << inst.N, dtype=torch.float64, device="cuda")
r = s.solve(tol=1e-13, max_iter=5000, pi=pi)
torch.cuda.synchronize()
t1 = time.time()
st = s.stats()
r2 = s.solve(tol=1e-13, max_iter=5000, pi=pi)
torch.cuda.synchronize()
t2 = time.time()
m = s.measures(pi)
print(json.dumps(dict(cfg=cfg, N=inst.N, rho=inst.rho, status=r["status"], iters=r["iters"], residual=r["residual"],
                      first_solve_s=t1 - t0, second_solve_s=t2 - t1, stats_first=st, stats=s.stats(),
                      loss=m["loss"], sum_pi=float(pi.sum()), min_pi=float(pi.min()),
                      mem_gb=torch.cuda.max_memory_allocated() / 1e9)))
