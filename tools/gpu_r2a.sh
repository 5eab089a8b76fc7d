#!/bin/bash
# round-2 session 2: tile-order A/B (group order vs chunked) at cfg4 / cfg5, parity spot check
cd "$(dirname "$0")/.."
HQ_ORDER=group HQ_GROUP_BITS=3 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "mid_sizes" > gpurun_out/r2a_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/r2a_parity.log
timeout 1500 python tools/env_ab.py 4 20 "chunk:" "g9:HQ_ORDER=group,HQ_GROUP_BITS=9" "g10:HQ_ORDER=group,HQ_GROUP_BITS=10" \
  "g11:HQ_ORDER=group,HQ_GROUP_BITS=11" "g11el:HQ_ORDER=group,HQ_GROUP_BITS=11,HQ_HPOL=0" "g11n:HQ_ORDER=group,HQ_GROUP_BITS=11,HQ_HPOL=1" > gpurun_out/r2a_ab4.log 2>&1
REPS=1 ROUNDS=1 timeout 1800 python tools/env_ab.py 5 12 "chunk:" "g10:HQ_ORDER=group,HQ_GROUP_BITS=10" \
  "g11:HQ_ORDER=group,HQ_GROUP_BITS=11" "g12:HQ_ORDER=group,HQ_GROUP_BITS=12" "g11n:HQ_ORDER=group,HQ_GROUP_BITS=11,HQ_HPOL=1" > gpurun_out/r2a_ab5.log 2>&1
echo done
