#!/bin/bash
# round-2 session 2: H-loop rewrite (3 rotating buffers, uniform L2 policies) + staged-body split
cd "$(dirname "$0")/.."
HQ_LOOP=host timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -q -x -k "not n31" > gpurun_out/r2d_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/r2d_parity.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "mid_sizes or device_loop" > gpurun_out/r2d_parity2.log 2>&1
echo "parity2 rc=$?" >> gpurun_out/r2d_parity2.log
timeout 600 python tools/env_ab.py 3 40 "main:" "base:HQ_LIB=$PWD/variants/libhq_base.so" > gpurun_out/r2d_ab3.log 2>&1
REPS=1 timeout 1500 python tools/env_ab.py 5 40 "main:" "base:HQ_LIB=$PWD/variants/libhq_base.so" "mainchunk:HQ_ORDER=chunk" > gpurun_out/r2d_ab5.log 2>&1
echo done
