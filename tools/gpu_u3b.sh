#!/bin/bash
# round-2 session 4: default bench, launch list, ncu --set full of one steady-state launch at cfg5 and cfg3
cd "$(dirname "$0")/.."
timeout 900 python bench.py > gpurun_out/u3_bench.json 2> gpurun_out/u3_bench.err; echo bench=$?
tail -c 2500 gpurun_out/u3_bench.json
timeout 300 python tools/prof_solve.py 3 150 > gpurun_out/u3_prof_plain3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/u3_launches_cfg3.csv python tools/prof_solve.py 3 150 > gpurun_out/u3_launch3.log 2>&1; echo list=$?
for c in 5 3; do
timeout 300 python tools/prof_solve.py $c 12 > gpurun_out/u3_prof_plain$c.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 10 -c 1 -o gpurun_out/u3_prof_cfg$c -f python tools/prof_solve.py $c 12 > gpurun_out/u3_ncu_full$c.log 2>&1; echo ncu$c=$?
ncu -i gpurun_out/u3_prof_cfg$c.ncu-rep --page details --csv > gpurun_out/u3_prof_cfg${c}_details.csv 2>/dev/null
ncu -i gpurun_out/u3_prof_cfg$c.ncu-rep --page raw --csv > gpurun_out/u3_prof_cfg${c}_raw.csv 2>/dev/null
ncu -i gpurun_out/u3_prof_cfg$c.ncu-rep --page source --csv --print-source sass > gpurun_out/u3_prof_cfg${c}_sass.csv 2>/dev/null
done
ls -la gpurun_out | head -40
