"""Per-instance precompute time (hq_stats[11]: rate programs, scatter weights) and a result
hash for library variants: python tools/time_precompute.py CFG NAME [NAME...] (GPU box;
variants/libhq_NAME.so).  Development aid."""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
child = r'''
import json, os, sys, hashlib
sys.path.insert(0, os.environ["ROOT"])
import torch, hqinst
from paper_2603_03019_b200 import hq
inst = hqinst.config_instance(int(os.environ["CFG"]))
out = []
for rep in range(3):
    s = hq.Solver.from_instance(inst)
    r = s.solve(tol=1e-13, max_iter=5000)
    st = s.stats()
    out.append(dict(precompute_ms=st["precompute_ms"], solve_ms=st["solve_ms"], iters=r["iters"],
                    pi_sha=hashlib.sha256(r["pi"].cpu().numpy().tobytes()).hexdigest()[:16]))
    s.close()
print(json.dumps(out))
'''
cfg = sys.argv[1]
for n in sys.argv[2:]:
    env = dict(os.environ, ROOT=ROOT, CFG=cfg, HQ_LIB=os.path.join(ROOT, "variants", f"libhq_{n}.so"))
    p = subprocess.run([sys.executable, "-c", child], env=env, capture_output=True, text=True, timeout=900)
    if p.returncode:
        print(n, "FAILED", p.stderr[-1500:])
        continue
    res = json.loads(p.stdout.strip().splitlines()[-1])
    print(json.dumps(dict(variant=n, precompute_ms=[round(x["precompute_ms"], 1) for x in res],
                          solve_ms=[round(x["solve_ms"], 1) for x in res], pi_sha=sorted({x["pi_sha"] for x in res}))))
