timeout 900 python tools/ab.py run ${CFG:-3} ${REPS:-4} $VARIANTS > gpurun_out/ab.log 2>&1; echo rc=$?; cat gpurun_out/ab.log | tail -12
