"""Throughput of the batched small-instance solver (row f2): instances/s for a batch shaped
like the paper's studies -- St. Paul-like N = 9 units, J = 71 atoms and Greenville-like
N = 6, J = 99, loads swept over 0.1..0.9 on seeded
synthetic geometries -- against the CPU oracle on a sample.  python tools/bench_batch.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hqinst  # noqa: E402
from paper_2603_03019_b200 import hq  # noqa: E402


def batch(N, J, B, seed0):
    insts = []
    for b in range(B):
        base = hqinst.generate(N, J, seed=seed0 + b // 9, rho=0.5)
        rho = 0.1 + 0.1 * (b % 9)
        lam = base.lam * (rho * base.mu.sum() / base.lam.sum())
        insts.append(hqinst.from_arrays(lam, base.mu, base.pref, rho=rho))
    return insts


out = {}
for (N, J, B) in [(9, 71, 1332), (6, 99, 1332), (11, 71, 1332), (12, 71, 592)]:
    insts = batch(N, J, B, 1000)
    lam = np.stack([i.lam for i in insts])
    mu = np.stack([i.mu for i in insts])
    pref = np.stack([i.pref for i in insts]).astype(np.int32)
    pi = torch.empty((B, 1 << N), dtype=torch.float64, device="cuda")
    hq.hq_batch_solve(lam, mu, pref, tol=1e-13, pi=pi, measures={})   # warm-up
    ts = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, it, res, st = hq.hq_batch_solve(lam, mu, pref, tol=1e-13, pi=pi, measures={})
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    rec = dict(N=N, J=J, B=B, seconds=t, instances_per_s=B / t, mean_sweeps=float(it.mean()),
               max_residual=float(res.max()), all_ok=bool((st == 0).all()))
    if "--cpu" in sys.argv:
        import oracle
        k = 27
        t0 = time.perf_counter()
        for inst in insts[:k]:
            oracle.solve(inst, tol=1e-13, max_iter=20000)
        tc = time.perf_counter() - t0
        rec["cpu_oracle_instances_per_s"] = k / tc
        rec["cpu_cores"] = oracle.num_threads()
    out[f"N{N}_J{J}"] = rec
    print(json.dumps(rec), flush=True)
