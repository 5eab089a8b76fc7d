#!/bin/bash
cd "$(dirname "$0")/.."
for cfg in 1 2; do
HQ_DEBUG_CTL=1 timeout 120 python -c "
import sys; sys.path.insert(0,'.')
import torch, hqinst
from paper_2603_03019_b200 import hq
inst = hqinst.config_instance($cfg)
s = hq.Solver.from_instance(inst)
for tol, mi in ((1e-13, 5000), (0.0, 40), (1e-13, 40)):
    try:
        r = s.solve(tol=tol, max_iter=mi); print(tol, mi, r['status'], r['iters'], r['residual'])
    except Exception as e: print(tol, mi, 'ERR', e)
" >> gpurun_out/s3c.log 2>&1
done
