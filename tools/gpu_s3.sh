#!/bin/bash
# round-2 session 3: first runs of the device-resident solve
cd "$(dirname "$0")/.."
TMO=120 timeout 300 python tools/dev_check.py 1 2 > gpurun_out/s3_dev12.log 2>&1
echo "dev12 rc=$?" >> gpurun_out/s3_dev12.log
grep -q FAILED gpurun_out/s3_dev12.log && exit 1
TMO=300 timeout 900 python tools/dev_check.py 3 4 > gpurun_out/s3_dev34.log 2>&1
TMO=600 REPS=2 timeout 1200 python tools/dev_check.py 5 > gpurun_out/s3_dev5.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_fullsize.py > gpurun_out/s3_tests.log 2>&1
echo done
