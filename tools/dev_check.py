"""Device-resident solve vs the host-looped path on BASELINE configs (development aid, GPU box):
python tools/dev_check.py CFG [CFG ...]  -> per config: iterations, residual, max |pi diff|,
solve / sweep times of both paths (each in a fresh process: HQ_LOOP is read at hq_create)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
child = r'''
import json, os, sys, time
sys.path.insert(0, os.environ["ROOT"])
import numpy as np, torch, hqinst
from paper_2603_03019_b200 import hq
cfg = int(os.environ["CFG"])
inst = hqinst.config_instance(cfg)
s = hq.Solver.from_instance(inst)
pi = torch.empty(1 << inst.N, dtype=torch.float64, device="cuda")
out = []
for rep in range(int(os.environ.get("REPS", "3"))):
    r = s.solve(tol=1e-13, max_iter=5000, pi=pi)
    st = s.stats()
    out.append(dict(status=r["status"], iters=r["iters"], residual=r["residual"], solve_ms=st["solve_ms"],
                    sweep_ms=st["sweep_ms"], halfsweeps=st["halfsweeps"], launches=st["launches"],
                    device_loop=st["device_loop"], kernel_ms=st["solve_kernel_ms"]))
np.save(os.environ["OUT"], pi.cpu().numpy())
print(json.dumps(out))
'''
for cfg in sys.argv[1:]:
    res = {}
    for loop in ("host", "device"):
        env = dict(os.environ, ROOT=ROOT, CFG=cfg, HQ_LOOP=loop, OUT=f"/tmp/pi_{cfg}_{loop}.npy")
        p = subprocess.run([sys.executable, "-c", child], env=env, capture_output=True, text=True,
                           timeout=int(os.environ.get("TMO", "600")))
        if p.returncode != 0:
            print(cfg, loop, "FAILED", p.stderr[-3000:], flush=True)
            continue
        res[loop] = json.loads(p.stdout.strip().splitlines()[-1])
    import numpy as np
    d = None
    if len(res) == 2:
        d = float(np.abs(np.load(f"/tmp/pi_{cfg}_host.npy") - np.load(f"/tmp/pi_{cfg}_device.npy")).max())
    print(json.dumps(dict(cfg=int(cfg), maxdiff=d, host=res.get("host"), device=res.get("device"))), flush=True)
