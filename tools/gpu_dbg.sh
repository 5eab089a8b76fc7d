timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
CFG=3 REPS=3 VARIANTS="rot hdr2" bash tools/gpu_ab.sh
CFG=4 REPS=2 VARIANTS="rot hdr2" bash tools/gpu_ab.sh
