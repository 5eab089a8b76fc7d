# large configs (cfg4 N=28, cfg5 N=31), each time-limited
timeout 400 python tools/run_cfg.py 4 > gpurun_out/run_cfg4.log 2>&1; echo cfg4 rc=$?; tail -c 1500 gpurun_out/run_cfg4.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
timeout 900 python tools/run_cfg.py 5 > gpurun_out/run_cfg5.log 2>&1; echo cfg5 rc=$?; tail -c 1500 gpurun_out/run_cfg5.log
