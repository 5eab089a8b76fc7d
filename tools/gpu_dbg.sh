# quick correctness/hang check (debug build with bounded mbarrier waits); every step time-limited
for cfg in 3 2; do
  timeout 90 python tools/prof_solve.py $cfg 12 > gpurun_out/dbg_cfg$cfg.log 2>&1; echo "cfg$cfg rc=$?"
  tail -c 400 gpurun_out/dbg_cfg$cfg.log; echo
done
timeout 300 python -m pytest tests -m gpu -x -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.log
