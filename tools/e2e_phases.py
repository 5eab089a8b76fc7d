"""Wall-clock phases of the end-to-end path bench.py times (create, solve incl. the
per-instance precompute, measures, device->host copies).  Development aid."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hqinst  # noqa: E402
from paper_2603_03019_b200 import hq  # noqa: E402

inst = hqinst.config_instance(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
host_pi = torch.empty(1 << inst.N, dtype=torch.float64).pin_memory()
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = hq.Solver.from_instance(inst)
    t1 = time.perf_counter()
    r = s.solve(tol=1e-13)
    t2 = time.perf_counter()
    m = s.measures(r["pi"])
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    host_pi.copy_(r["pi"])
    w = m["workload"].cpu()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    st = s.stats()
    s.close()
    t5 = time.perf_counter()
    print(f"create {1e3*(t1-t0):7.1f}  solve {1e3*(t2-t1):7.1f} (precompute {st['precompute_ms']:.1f}, "
          f"solve events {st['solve_ms']:.1f})  measures {1e3*(t3-t2):6.1f}  d2h {1e3*(t4-t3):6.1f}  "
          f"close {1e3*(t5-t4):6.1f}  total {1e3*(t5-t0):7.1f} ms")
