#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python tools/ab.py run 3 3 r1 main@HQ_LOOP=host nortab@HQ_LOOP=host > gpurun_out/s9_ab3.log 2>&1
timeout 900 python tools/ab.py run 4 2 r1 main nortab > gpurun_out/s9_ab4.log 2>&1
echo done
