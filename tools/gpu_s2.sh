#!/bin/bash
# round-2 session 2: program statistics, chunk-size A/B, ncu of the cfg5 sweep kernel
cd "$(dirname "$0")/.."
timeout 300 python tools/prog_stats.py 3 > gpurun_out/s2_prog3.json 2> gpurun_out/s2_prog3.err
timeout 600 python tools/prog_stats.py 5 > gpurun_out/s2_prog5.json 2> gpurun_out/s2_prog5.err
timeout 900 python tools/ab.py run 4 2 main@HQ_CHUNK_BITS=5 main@HQ_CHUNK_BITS=6 main@HQ_CHUNK_BITS=7 main@HQ_CHUNK_BITS=8 > gpurun_out/s2_ab4.log 2>&1
RHO=0.6 timeout 1500 python tools/ab.py run 5 1 main@HQ_CHUNK_BITS=5 main@HQ_CHUNK_BITS=7 > gpurun_out/s2_ab5.log 2>&1
timeout 300 python tools/prof_solve.py 5 30 > gpurun_out/s2_plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep3 -s 40 -c 1 -o gpurun_out/s2_prof_cfg5 -f python tools/prof_solve.py 5 30 > gpurun_out/s2_ncu5.log 2>&1
echo done
