#!/bin/bash
cd "$(dirname "$0")/.."
REPS=1 timeout 2400 python tools/env_ab.py 5 40 "main:" "inN:HQ_INPOL=1" "inH:HQ_INPOL=3" "pfout:HQ_PFMIN=11" "inNpfout:HQ_INPOL=1,HQ_PFMIN=11" "g12inN:HQ_GROUP_BITS=12,HQ_INPOL=1" "g10inH:HQ_GROUP_BITS=10,HQ_INPOL=3" > gpurun_out/r2i_ab5.log 2>&1
timeout 900 python tools/env_ab.py 4 40 "main:" "inN:HQ_INPOL=1" "inH:HQ_INPOL=3" "pfout:HQ_PFMIN=11" > gpurun_out/r2i_ab4.log 2>&1
timeout 600 python tools/env_ab.py 3 40 "main:" "inN:HQ_INPOL=1" "inH:HQ_INPOL=3" > gpurun_out/r2i_ab3.log 2>&1
echo done
