#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_buffer.py tests/test_gpu_response.py tests/test_gpu_batch.py tests/test_gpu_fullsize.py -k "not cfg3_whole and not cfg4 and not cfg5 and not mid_sizes" -q -x > gpurun_out/r2l_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2l_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2l_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2l_smoke.log
echo done
