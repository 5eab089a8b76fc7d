#!/bin/bash
# round-2 session 1: GPU tests on the modified library, tile-order A/B at cfg4 / cfg5
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s1_smi.txt
free -g > gpurun_out/s1_free.txt; nproc >> gpurun_out/s1_free.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s1_tests.log 2>&1
timeout 900 python tools/ab.py run 4 2 main@HQ_ORDER=popcount main@HQ_ORDER=chunk main@HQ_ORDER=chunk@HQ_CHUNK_BITS=1 main@HQ_ORDER=chunk@HQ_CHUNK_BITS=5 > gpurun_out/s1_ab4.log 2>&1
RHO=0.6 timeout 1200 python tools/ab.py run 5 1 main@HQ_ORDER=popcount main@HQ_ORDER=chunk > gpurun_out/s1_ab5.log 2>&1
