"""Compare the scalar block after K half-sweeps of the host-looped and the device-resident solve
(development aid, GPU box): python tools/dev_debug.py CFG SWEEPS"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
child = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"])
import numpy as np, torch, hqinst
from paper_2603_03019_b200 import hq
inst = hqinst.config_instance(int(os.environ["CFG"]))
s = hq.Solver.from_instance(inst)
pi = torch.empty(1 << inst.N, dtype=torch.float64, device="cuda")
try:
    r = s.solve(tol=0.0, max_iter=int(os.environ["SW"]), pi=pi)
    print("status", r["status"], r["iters"], r["residual"])
except Exception as e:
    print("ERR", e)
blk = hq.hq_debug_copy(s.h, 0, 8 * 416, np.float64)
np.save(os.environ["OUT"], blk)
print(s.stats())
'''
cfg, sw = sys.argv[1], sys.argv[2]
import numpy as np
for loop in ("host", "device"):
    env = dict(os.environ, ROOT=ROOT, CFG=cfg, SW=sw, HQ_LOOP=loop, OUT=f"/tmp/blk_{loop}.npy")
    p = subprocess.run([sys.executable, "-c", child], env=env, capture_output=True, text=True, timeout=300)
    print(loop, p.stdout[-1500:], p.stderr[-1500:])
a, b = np.load("/tmp/blk_host.npy"), np.load("/tmp/blk_device.npy")
names = ["LAM", "MU", "ALPHA", "BETA", "PN", "OM", "KA", "DL1", "SUMP", "RNUM", "RDEN", "MUSTAR", "MISC"]
offs = [0, 32, 64, 96, 128, 176, 208, 240, 272, 304, 336, 368, 400]
for n, o in zip(names, offs):
    print(n, "host  ", np.array2string(a[o:o + 16], precision=6, max_line_width=250))
    print(n, "device", np.array2string(b[o:o + 16], precision=6, max_line_width=250))
