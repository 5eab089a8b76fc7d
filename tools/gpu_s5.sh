#!/bin/bash
# ncu: k_loop3 (device loop, whole cfg3 solve, 40 sweeps) vs k_sweep3 (host loop, one steady-state launch)
cd "$(dirname "$0")/.."
timeout 300 python tools/prof_dev.py 3 40 > gpurun_out/s5_plain_dev.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_loop3 -c 1 -o gpurun_out/s5_loop3_cfg3 -f python tools/prof_dev.py 3 40 > gpurun_out/s5_ncu_dev.log 2>&1
HQ_LOOP=host timeout 300 python tools/prof_dev.py 3 40 > gpurun_out/s5_plain_host.log 2>&1 && \
HQ_LOOP=host timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep3 -s 60 -c 1 -o gpurun_out/s5_sweep3_cfg3 -f python tools/prof_dev.py 3 40 > gpurun_out/s5_ncu_host.log 2>&1
echo done
