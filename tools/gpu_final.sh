# round deliverable measurements (each step time-limited); profiles are copied to profiles/ afterwards
nproc; lscpu | grep -E "Model name|^CPU\(s\)" | head -2
( time timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err ) 2>&1 | tail -3; echo bench=$?
tail -c 2500 gpurun_out/bench_default.json
( time timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err ) 2>&1 | tail -3
cat gpurun_out/bench_reference.json
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu_list=$?
timeout 120 python tools/prof_solve.py 3 30 > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep3 -s 40 -c 1 -o gpurun_out/prof_cfg3 -f python tools/prof_solve.py 3 30 > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
