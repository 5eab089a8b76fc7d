#!/bin/bash
# round-2 session 4: full GPU suite on the final library
cd "$(dirname "$0")/.."
free -g | head -2; nproc
timeout 3300 python -m pytest tests -m gpu -q -x --timeout 900 --durations=15 > gpurun_out/u3_pytest_gpu.log 2>&1; echo pytest=$?
tail -25 gpurun_out/u3_pytest_gpu.log
