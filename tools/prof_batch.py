"""Profiling driver for the batched solver (row f2): one call on a St. Paul-sized batch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import hqinst  # noqa: E402
from paper_2603_03019_b200 import hq  # noqa: E402

insts = [hqinst.generate(9, 71, seed=1000 + b // 9, rho=0.1 + 0.1 * (b % 9)) for b in range(1332)]
args = (np.stack([i.lam for i in insts]), np.stack([i.mu for i in insts]), np.stack([i.pref for i in insts]))
hq.hq_batch_solve(*args, tol=1e-13, measures={})
hq.hq_batch_solve(*args, tol=1e-13, measures={})
