#!/bin/bash
cd "$(dirname "$0")/.."
V=$PWD/variants
python - > gpurun_out/r2f_dbg.log 2>&1 <<'PY'
import sys, json
sys.path.insert(0, ".")
import torch, hqinst
from paper_2603_03019_b200 import hq
for cfg in (3,):
    inst = hqinst.config_instance(cfg)
    s = hq.Solver.from_instance(inst)
    try:
        r = s.solve(tol=1e-13, max_iter=5000)
        print(cfg, r["status"], r["iters"], r["residual"], s.stats()["sweep_ms"])
    except Exception as e:
        print(cfg, "ERR", e)
PY
HQ_LOOP=host timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2f_parity.log 2>&1
timeout 900 python tools/env_ab.py 3 40 "main:" "pfo:HQ_PFO=1" "pfh4:HQ_PFH=4" "pfh6:HQ_PFH=6" "hbuf2:HQ_LIB=$V/libhq_hbuf2.so" > gpurun_out/r2f_ab3.log 2>&1
REPS=1 timeout 1800 python tools/env_ab.py 5 40 "main:" "pfo:HQ_PFO=1" "pfh4:HQ_PFH=4" "pfh6:HQ_PFH=6" "pfh6o:HQ_PFH=6,HQ_PFO=1" "hbuf2:HQ_LIB=$V/libhq_hbuf2.so" > gpurun_out/r2f_ab5.log 2>&1
echo done
