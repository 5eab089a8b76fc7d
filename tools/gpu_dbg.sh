for cfg in 1 2 3; do
  timeout 60 python tools/prof_solve.py $cfg 3 > gpurun_out/dbg_cfg$cfg.log 2>&1; echo "cfg$cfg rc=$?"; tail -c 300 gpurun_out/dbg_cfg$cfg.log; echo
done
timeout 200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 60 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
