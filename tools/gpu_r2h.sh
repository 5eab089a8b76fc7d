#!/bin/bash
cd "$(dirname "$0")/.."
V=$PWD/variants
timeout 600 python tools/env_ab.py 3 40 "main:" "lastwarp:HQ_LIB=$V/libhq_lastwarp.so" > gpurun_out/r2h_ab3.log 2>&1
REPS=1 timeout 1200 python tools/env_ab.py 5 40 "main:" "lastwarp:HQ_LIB=$V/libhq_lastwarp.so" > gpurun_out/r2h_ab5.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sweep3 -s 70 -c 1 -o gpurun_out/r2h_prof_cfg5 -f python tools/prof_solve.py 5 40 > gpurun_out/r2h_ncu5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep3 -s 60 -c 1 -o gpurun_out/r2h_prof_cfg3 -f python tools/prof_solve.py 3 40 > gpurun_out/r2h_ncu3.log 2>&1
echo done
