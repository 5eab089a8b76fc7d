timeout 120 python tools/check_programs.py 12 40 0 4 > gpurun_out/chk12.log 2>&1; echo rc=$?; tail -12 gpurun_out/chk12.log
timeout 120 python tools/check_programs.py 13 40 5 4 > gpurun_out/chk13.log 2>&1; echo rc=$?; tail -12 gpurun_out/chk13.log
