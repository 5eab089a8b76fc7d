timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/prof_solve.py 2 1 > gpurun_out/memcheck.log 2>&1; echo rc=$?
head -60 gpurun_out/memcheck.log
