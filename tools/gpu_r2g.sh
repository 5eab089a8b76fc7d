#!/bin/bash
cd "$(dirname "$0")/.."
HQ_LOOP=host timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -k "not n31" > gpurun_out/r2g_parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2g_parity.log
timeout 600 python tools/env_ab.py 3 40 "main:" "pfh3:HQ_PFH=3" > gpurun_out/r2g_ab3.log 2>&1
timeout 900 python tools/env_ab.py 4 40 "main:" "pfh3:HQ_PFH=3" "pfh5:HQ_PFH=5" "nopf:HQ_PFH=0,HQ_PFO=0" > gpurun_out/r2g_ab4.log 2>&1
REPS=1 timeout 1800 python tools/env_ab.py 5 40 "main:" "pfh3:HQ_PFH=3" "pfh5:HQ_PFH=5" "pfh4no:HQ_PFO=0" "g10:HQ_GROUP_BITS=10" "g12:HQ_GROUP_BITS=12" > gpurun_out/r2g_ab5.log 2>&1
echo done
