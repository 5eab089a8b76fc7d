#!/bin/bash
cd "$(dirname "$0")/.."
REPS=1 timeout 2400 python tools/env_ab.py 5 40 "main:" "p40:HQ_PERSIST_MB=40" "p80:HQ_PERSIST_MB=80" "p80g10:HQ_PERSIST_MB=80,HQ_GROUP_BITS=10" > gpurun_out/r2j_ab5.log 2>&1
echo done
