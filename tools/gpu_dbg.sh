timeout 300 python tools/check_programs.py 19 40 0 2 > gpurun_out/chk.log 2>&1; echo rc=$?; tail -12 gpurun_out/chk.log
