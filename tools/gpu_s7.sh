#!/bin/bash
# round-2 session 7: full GPU suite (incl. full-size parity), bench (cfg5 headline + cfg3), ncu of cfg5
cd "$(dirname "$0")/.."
nproc > gpurun_out/s7_env.txt; free -g >> gpurun_out/s7_env.txt
timeout 3000 python -m pytest tests -m gpu -q -x --durations=30 > gpurun_out/s7_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/s7_tests.log
timeout 1800 python bench.py > gpurun_out/s7_bench.json 2> gpurun_out/s7_bench.err
echo "bench rc=$?" >> gpurun_out/s7_bench.err
timeout 300 python tools/prof_solve.py 5 30 > gpurun_out/s7_plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep3 -s 40 -c 1 -o gpurun_out/s7_prof_cfg5 -f python tools/prof_solve.py 5 30 > gpurun_out/s7_ncu5.log 2>&1
echo done
