# ncu capture of the sweep kernel (run under gpurun from the repo root)
CFG=${1:-3}
timeout 120 python tools/prof_solve.py $CFG 12 > gpurun_out/prof_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$CFG.csv python tools/prof_solve.py $CFG 12 > gpurun_out/ncu_launch.log 2>&1 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 10 -c 1 -o gpurun_out/prof_cfg$CFG -f python tools/prof_solve.py $CFG 12 > gpurun_out/ncu_full.log 2>&1
echo rc=$?
