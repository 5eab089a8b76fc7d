#!/bin/bash
# round-2 session 2: group order at cfg3 (round-robin popcount order), cfg5 steady state, ncu of cfg5 g11
cd "$(dirname "$0")/.."
timeout 900 python tools/env_ab.py 3 40 "pop:" "rr:HQ_ORDER=group,HQ_GROUP_BITS=11" "g8:HQ_ORDER=group,HQ_GROUP_BITS=8" "g9:HQ_ORDER=group,HQ_GROUP_BITS=9" > gpurun_out/r2b_ab3.log 2>&1
REPS=1 ROUNDS=1 timeout 1200 python tools/env_ab.py 5 40 "chunk:" "g11:HQ_ORDER=group,HQ_GROUP_BITS=11" "g11el:HQ_ORDER=group,HQ_GROUP_BITS=11,HQ_HPOL=0" > gpurun_out/r2b_ab5.log 2>&1
HQ_ORDER=group HQ_GROUP_BITS=11 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sweep3 -s 70 -c 1 -o gpurun_out/r2b_prof_cfg5_g11 -f python tools/prof_solve.py 5 40 > gpurun_out/r2b_ncu5.log 2>&1
echo done
