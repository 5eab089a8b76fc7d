#!/bin/bash
# round-2 session 2: L2 prefetch of the next tile's outer neighbour blocks (group order)
cd "$(dirname "$0")/.."
REPS=1 timeout 1500 python tools/env_ab.py 5 40 "g11pf:HQ_ORDER=group,HQ_GROUP_BITS=11" "g11nopf:HQ_ORDER=group,HQ_GROUP_BITS=11,HQ_PF=32" "g11pf0:HQ_ORDER=group,HQ_GROUP_BITS=11,HQ_PF=0" "g10pf:HQ_ORDER=group,HQ_GROUP_BITS=10" "g12pf:HQ_ORDER=group,HQ_GROUP_BITS=12" > gpurun_out/r2c_ab5.log 2>&1
timeout 900 python tools/env_ab.py 4 40 "g11pf:HQ_ORDER=group,HQ_GROUP_BITS=11" "g11nopf:HQ_ORDER=group,HQ_GROUP_BITS=11,HQ_PF=32" "g11pf0:HQ_ORDER=group,HQ_GROUP_BITS=11,HQ_PF=0" "g9pf:HQ_ORDER=group,HQ_GROUP_BITS=9" > gpurun_out/r2c_ab4.log 2>&1
timeout 600 python tools/env_ab.py 3 40 "pop:" "pf0:HQ_PF=0" > gpurun_out/r2c_ab3.log 2>&1
echo done
