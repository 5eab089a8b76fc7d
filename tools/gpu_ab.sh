# same-box A/B of library variants (tools/ab.py); log per config
timeout 900 python tools/ab.py run ${CFG:-3} ${REPS:-4} $VARIANTS > gpurun_out/ab_cfg${CFG:-3}.log 2>&1; echo rc=$?; tail -12 gpurun_out/ab_cfg${CFG:-3}.log
