timeout 900 python -m pytest tests -m gpu -q --timeout 400 --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -25 gpurun_out/pytest_gpu.log
