#!/bin/bash
cd "$(dirname "$0")/.."
timeout 300 python tools/dev_debug.py 1 1 > gpurun_out/s3b_dbg.log 2>&1
timeout 300 python tools/dev_debug.py 2 3 >> gpurun_out/s3b_dbg.log 2>&1
bash tools/gpu_s3.sh
