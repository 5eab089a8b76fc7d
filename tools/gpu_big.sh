timeout 900 python -m pytest tests -m gpu -q --timeout 400 --durations=6 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -12 gpurun_out/pytest_gpu.log
timeout 600 python tools/run_cfg.py 5 > gpurun_out/run_cfg5.log 2>&1; echo cfg5 rc=$?; tail -c 1200 gpurun_out/run_cfg5.log
