"""A/B timing of library variants on the same GPU, interleaved.

  python tools/ab.py build NAME [DEFINE ...]     (here: compile variants/libhq_NAME.so)
  python tools/ab.py run CFG REPS NAME [NAME...] (GPU box: time hq_solve per variant)

Each run creates a solver per variant, warms it up, then alternates variants for REPS
rounds; prints the median solve time and sweep-kernel time of each.  Development aid."""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VAR = os.path.join(ROOT, "variants")

if sys.argv[1] == "build":
    sys.path.insert(0, ROOT)
    from paper_2603_03019_b200 import build as b

    os.makedirs(VAR, exist_ok=True)
    b.build(out=os.path.join(VAR, f"libhq_{sys.argv[2]}.so"), defines=sys.argv[3:])
    sys.exit(0)

cfg, reps, names = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4:]
child = r'''
import json, os, statistics, sys
sys.path.insert(0, os.environ["ROOT"])
import torch, hqinst
from paper_2603_03019_b200 import hq
inst = hqinst.config_instance(int(os.environ["CFG"]), rho=float(os.environ["RHO"]) if os.environ.get("RHO") else None)
s = hq.Solver.from_instance(inst)
pi = torch.empty(1 << inst.N, dtype=torch.float64, device="cuda")
for _ in range(2):
    s.solve(tol=1e-13, max_iter=5000, pi=pi)
out = []
for _ in range(int(os.environ["REPS"])):
    r = s.solve(tol=1e-13, max_iter=5000, pi=pi)
    st = s.stats()
    out.append((st["solve_ms"], st["sweep_ms"], r["iters"], r["residual"], st.get("program_nwv", -1),
                st.get("chunk_bits", -1), 0))
print(json.dumps(out))
'''
res = {n: [] for n in names}
for rnd in range(2):   # two interleaved rounds of fresh processes
    for n in names:
        # NAME@cta / NAME@warp forces the program granularity; NAME@VAR=VALUE sets an env var
        lib, *mods = n.split("@")
        libpath = os.path.join(ROOT, "paper_2603_03019_b200", "libhq.so") if lib == "main" else \
            os.path.join(VAR, f"libhq_{lib}.so")
        env = dict(os.environ, ROOT=ROOT, CFG=str(cfg), REPS=str(reps), HQ_LIB=libpath)
        for mod in mods:
            k, eq, v = mod.partition("=")
            if eq:
                env[k] = v
            else:
                env["HQ_PROG"] = mod
        p = subprocess.run([sys.executable, "-c", child], env=env, capture_output=True, text=True, timeout=600)
        if p.returncode != 0:
            print(n, "FAILED", p.stderr[-2000:])
            continue
        res[n] += json.loads(p.stdout.strip().splitlines()[-1])
for n in names:
    if not res[n]:
        continue
    solve = statistics.median(x[0] for x in res[n])
    sweep = statistics.median(x[1] for x in res[n])
    x = res[n][0]
    print(json.dumps(dict(variant=n, solve_ms=round(solve, 2), sweep_ms=round(sweep, 2), iters=x[2],
                          residual=x[3], samples=len(res[n]), prog_nwv=x[4] if len(x) > 4 else None,
                          tune_ms=(x[5], x[6]) if len(x) > 6 else None)))
