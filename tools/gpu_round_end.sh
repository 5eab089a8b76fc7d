# round-end measurements: bench (default + reference arm), cfg2/cfg4/cfg5 solves, ncu launch list
( time timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err ) 2>&1 | tail -3; echo bench=$?
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo ref=$?
for c in 2 4 5; do timeout 900 python tools/run_cfg.py $c > gpurun_out/run_cfg$c.json 2> gpurun_out/run_cfg$c.err; echo cfg$c=$?; done
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu_list=$?
