#!/bin/bash
# round-2 session 2: full GPU suite, bench, launch list and ncu of the current kernel
cd "$(dirname "$0")/.."
timeout 3000 python -m pytest tests -m gpu -q -x --durations=20 > gpurun_out/r2k_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2k_tests.log
timeout 1800 python bench.py > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err
echo "bench rc=$?" >> gpurun_out/r2k_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2k_launches_cfg3.csv python tools/prof_solve.py 3 150 > gpurun_out/r2k_launch3.log 2>&1
echo done
