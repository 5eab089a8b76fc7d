#!/bin/bash
# round-2 session 4, final measurements: 8-warp-CTA A/B, ncu --set full of one steady-state launch
# (cfg5, cfg3; the summary bench.py reads is regenerated on the box), launch list, default bench
cd "$(dirname "$0")/.."
V=/root/repo/variants
# the GPU tests the u4 run did not reach (it stopped at the group-lag test's stale default), and the
# parity cases that exercise the sweep kernel, on the final library (tile-unit slices consumed in place)
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_large.py tests/test_gpu_parity.py tests/test_gpu_response.py tests/test_gpu_buffer.py -q --timeout 900 --durations=8 -k "not cfg5 and not cfg3_whole and not n28_iterates" > gpurun_out/u5_pytest_rest.log 2>&1; echo pytest_rest=$?
tail -14 gpurun_out/u5_pytest_rest.log
ROUNDS=2 REPS=2 timeout 400 python tools/env_ab.py 3 60 main: nw3:HQ_LIB=$V/libhq_nw3.so,HQ_NW=3 > gpurun_out/u5_ab_nw3_cfg3.jsonl 2>&1; echo abn3=$?
cat gpurun_out/u5_ab_nw3_cfg3.jsonl
ROUNDS=1 REPS=2 timeout 600 python tools/env_ab.py 5 20 main: nw3g12:HQ_LIB=$V/libhq_nw3.so,HQ_NW=3,HQ_GROUP_BITS=12 nw3g11:HQ_LIB=$V/libhq_nw3.so,HQ_NW=3 > gpurun_out/u5_ab_nw3_cfg5.jsonl 2>&1; echo abn5=$?
cat gpurun_out/u5_ab_nw3_cfg5.jsonl
for c in 5 3; do
timeout 300 python tools/prof_solve.py $c 24 > gpurun_out/u5_prof_plain$c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep3 -s 40 -c 1 -o gpurun_out/u5_prof_cfg$c -f python tools/prof_solve.py $c 24 > gpurun_out/u5_ncu_full$c.log 2>&1; echo ncu$c=$?
ncu -i gpurun_out/u5_prof_cfg$c.ncu-rep --page details --csv > gpurun_out/u5_prof_cfg${c}_details.csv 2>/dev/null
ncu -i gpurun_out/u5_prof_cfg$c.ncu-rep --page source --csv --print-source sass > gpurun_out/u5_prof_cfg${c}_sass.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/u5_prof_cfg$c.ncu-rep $c > gpurun_out/u5_ncu_summary_cfg$c.json 2>&1
done
cp profiles/ncu_summary.json gpurun_out/u5_ncu_summary.json
timeout 300 python tools/prof_solve.py 3 150 > gpurun_out/u5_prof_plain3b.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/u5_launches_cfg3.csv python tools/prof_solve.py 3 150 > gpurun_out/u5_launch3.log 2>&1; echo list=$?
timeout 1200 python bench.py > gpurun_out/u5_bench.json 2> gpurun_out/u5_bench.err; echo bench=$?
tail -c 3000 gpurun_out/u5_bench.json
rm -f gpurun_out/u5_prof_cfg5.ncu-rep   # keep the pull below 64 MiB (summaries above are what is committed)
ls -la gpurun_out | head -40
