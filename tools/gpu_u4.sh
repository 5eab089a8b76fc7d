#!/bin/bash
# round-2 session 4: A/B of the tile-unit buffer schemes on the compact kernel, then the full GPU suite
cd "$(dirname "$0")/.."
V=/root/repo/variants
timeout 600 python tools/ab.py run 3 3 main nocompact h1 h2 h4 base > gpurun_out/u4_ab_cfg3.log 2>&1; echo ab3=$?
cat gpurun_out/u4_ab_cfg3.log
ROUNDS=2 REPS=2 timeout 1200 python tools/env_ab.py 5 20 main: lag0:HQ_GLAG=0 lag1:HQ_GLAG=1 lag3:HQ_GLAG=3 h1:HQ_LIB=$V/libhq_h1.so h2:HQ_LIB=$V/libhq_h2.so h4:HQ_LIB=$V/libhq_h4.so g10:HQ_GROUP_BITS=10 base:HQ_LIB=$V/libhq_base.so > gpurun_out/u4_ab_cfg5.jsonl 2>&1; echo ab5=$?
cat gpurun_out/u4_ab_cfg5.jsonl
ROUNDS=2 REPS=2 timeout 600 python tools/env_ab.py 4 40 main: lag2:HQ_GLAG=2 h1:HQ_LIB=$V/libhq_h1.so h2:HQ_LIB=$V/libhq_h2.so h4:HQ_LIB=$V/libhq_h4.so base:HQ_LIB=$V/libhq_base.so > gpurun_out/u4_ab_cfg4.jsonl 2>&1; echo ab4=$?
cat gpurun_out/u4_ab_cfg4.jsonl
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 --durations=12 > gpurun_out/u4_pytest_gpu.log 2>&1; echo pytest=$?
tail -22 gpurun_out/u4_pytest_gpu.log
