#!/bin/bash
# fast flush: parity smoke + A/B against the round-1 library + chunk-size A/B at cfg4 / cfg5
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -q -x > gpurun_out/s8_tests.log 2>&1
timeout 900 python tools/ab.py run 3 3 r1 main@HQ_LOOP=host main@HQ_LOOP=device > gpurun_out/s8_ab3.log 2>&1
timeout 900 python tools/ab.py run 4 2 main@HQ_CHUNK_BITS=5 main@HQ_CHUNK_BITS=0 main@HQ_CHUNK_BITS=2 > gpurun_out/s8_ab4.log 2>&1
RHO=0.6 timeout 1800 python tools/ab.py run 5 1 main@HQ_CHUNK_BITS=5 main@HQ_CHUNK_BITS=0 main@HQ_CHUNK_BITS=2 > gpurun_out/s8_ab5.log 2>&1
echo done
