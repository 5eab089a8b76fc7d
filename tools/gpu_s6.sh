#!/bin/bash
cd "$(dirname "$0")/.."
TMO=300 timeout 900 python tools/dev_check.py 2 3 > gpurun_out/s6_dev.log 2>&1
