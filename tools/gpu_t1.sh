#!/bin/bash
# round-2 session 3: verify HEAD (k_sweep2 retired) -- GPU suite + default bench
cd "$(dirname "$0")/.."
nproc
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 --durations=15 > gpurun_out/t1_pytest_gpu.log 2>&1; echo pytest=$?
tail -25 gpurun_out/t1_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/t1_bench.json 2> gpurun_out/t1_bench.err; echo bench=$?
tail -c 1500 gpurun_out/t1_bench.json
