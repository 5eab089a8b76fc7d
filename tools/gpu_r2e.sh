#!/bin/bash
# round-2 session 2: which part of the H-loop rewrite costs time; layout microbenchmark
cd "$(dirname "$0")/.."
V=$PWD/variants
timeout 300 tools/layout_ab/layout_ab 24 10 > gpurun_out/r2e_layout.log 2>&1
timeout 300 tools/layout_ab/layout_ab 28 5 >> gpurun_out/r2e_layout.log 2>&1
timeout 900 python tools/env_ab.py 3 40 "main:" "nosplit:HQ_LIB=$V/libhq_nosplit.so" "hbuf2:HQ_LIB=$V/libhq_hbuf2.so" "hbuf2nosplit:HQ_LIB=$V/libhq_hbuf2nosplit.so" "base:HQ_LIB=$V/libhq_base.so" > gpurun_out/r2e_ab3.log 2>&1
REPS=1 timeout 1800 python tools/env_ab.py 5 40 "main:" "nosplit:HQ_LIB=$V/libhq_nosplit.so" "hbuf2:HQ_LIB=$V/libhq_hbuf2.so" "hbuf2nosplit:HQ_LIB=$V/libhq_hbuf2nosplit.so" > gpurun_out/r2e_ab5.log 2>&1
echo done
