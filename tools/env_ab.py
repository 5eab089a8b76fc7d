"""Same-box A/B of environment switches (tile order, loop, ...) on a fixed number of sweeps.

  python tools/env_ab.py CFG SWEEPS [RHO=..] VARIANT [VARIANT ...]
  VARIANT = "label:K=V,K2=V2" (env vars read at hq_create); "label:" = defaults

Each variant runs in a fresh process, twice (interleaved): create, one warm-up solve of
SWEEPS sweeps (tol = 0), then REPS timed solves.  Prints per variant the median sweep-kernel
time per half-sweep and per solve.  Development aid (GPU box)."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
child = r'''
import json, os, sys
sys.path.insert(0, os.environ["ROOT"])
import torch, hqinst
from paper_2603_03019_b200 import hq
rho = os.environ.get("RHO")
inst = hqinst.config_instance(int(os.environ["CFG"]), rho=float(rho) if rho else None)
s = hq.Solver.from_instance(inst)
pi = torch.empty(1 << inst.N, dtype=torch.float64, device="cuda")
sw = int(os.environ["SWEEPS"])
s.solve(tol=0.0, max_iter=sw, pi=pi)
out = []
for _ in range(int(os.environ.get("REPS", "2"))):
    r = s.solve(tol=0.0, max_iter=sw, pi=pi)
    st = s.stats()
    out.append(dict(solve_ms=st["solve_ms"], sweep_ms=st["sweep_ms"], hs=st["halfsweeps"], res=r["residual"],
                    chunk_bits=st.get("chunk_bits")))
print(json.dumps(out))
'''
cfg, sweeps = sys.argv[1], sys.argv[2]
args = sys.argv[3:]
rho = None
if args and args[0].startswith("RHO="):
    rho = args.pop(0)[4:]
variants = []
for v in args:
    label, _, kv = v.partition(":")
    env = dict(x.split("=", 1) for x in kv.split(",") if x)
    variants.append((label, env))
res = {lab: [] for lab, _ in variants}
for rnd in range(int(os.environ.get("ROUNDS", "2"))):
    for lab, e in variants:
        env = dict(os.environ, ROOT=ROOT, CFG=cfg, SWEEPS=sweeps, **e)
        if rho:
            env["RHO"] = rho
        p = subprocess.run([sys.executable, "-c", child], env=env, capture_output=True, text=True,
                           timeout=int(os.environ.get("TMO", "900")))
        if p.returncode != 0:
            print(lab, "FAILED", p.stderr[-2000:], flush=True)
            continue
        res[lab] += json.loads(p.stdout.strip().splitlines()[-1])
for lab, _ in variants:
    if not res[lab]:
        continue
    sw = statistics.median(x["sweep_ms"] for x in res[lab])
    so = statistics.median(x["solve_ms"] for x in res[lab])
    hs = res[lab][0]["hs"]
    print(json.dumps(dict(variant=lab, cfg=cfg, sweeps=sweeps, solve_ms=round(so, 2), sweep_ms=round(sw, 2),
                          ms_per_halfsweep=round(sw / max(hs, 1), 4), samples=len(res[lab]),
                          residual=res[lab][0]["res"], chunk_bits=res[lab][0]["chunk_bits"])), flush=True)
