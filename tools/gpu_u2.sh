#!/bin/bash
# round-2 session 4: leaner tile-unit loop (compile-time nW, resolved L2 policies, paired
# prefetch, 64-bit bases in the epilogue): parity subset, same-box A/B, source-level ncu
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_large.py tests/test_gpu_parity.py -q -x --timeout 600 -k "mid_sizes or tile_orders or cfg3_against or cfg3_bitwise or iterates or cfg4_truncated" > gpurun_out/u2_pytest.log 2>&1; echo pytest=$?
tail -4 gpurun_out/u2_pytest.log
timeout 900 python tools/ab.py run 3 3 main m3 m2 m1 base hbuf3 compact h1 hbuf3c > gpurun_out/u2_ab_cfg3.log 2>&1; echo ab3=$?
cat gpurun_out/u2_ab_cfg3.log
V=/root/repo/variants
ROUNDS=2 REPS=2 timeout 1700 python tools/env_ab.py 5 20 main: m3:HQ_LIB=$V/libhq_m3.so m2:HQ_LIB=$V/libhq_m2.so m1:HQ_LIB=$V/libhq_m1.so base:HQ_LIB=$V/libhq_base.so hbuf3:HQ_LIB=$V/libhq_hbuf3.so compact:HQ_LIB=$V/libhq_compact.so h1:HQ_LIB=$V/libhq_h1.so hbuf3c:HQ_LIB=$V/libhq_hbuf3c.so pf2:HQ_PFH=2 pf3:HQ_PFH=3 pf6:HQ_PFH=6 pf0:HQ_PFH=0 lag2:HQ_GLAG=2 > gpurun_out/u2_ab_cfg5.jsonl 2>&1; echo ab5=$?
cat gpurun_out/u2_ab_cfg5.jsonl
ROUNDS=2 REPS=2 timeout 600 python tools/env_ab.py 4 40 main: m3:HQ_LIB=$V/libhq_m3.so m2:HQ_LIB=$V/libhq_m2.so m1:HQ_LIB=$V/libhq_m1.so base:HQ_LIB=$V/libhq_base.so hbuf3:HQ_LIB=$V/libhq_hbuf3.so compact:HQ_LIB=$V/libhq_compact.so h1:HQ_LIB=$V/libhq_h1.so hbuf3c:HQ_LIB=$V/libhq_hbuf3c.so > gpurun_out/u2_ab_cfg4.jsonl 2>&1; echo ab4=$?
cat gpurun_out/u2_ab_cfg4.jsonl
# source-level profile of one steady-state launch at cfg3 (after the plain run exits 0)
timeout 120 python tools/prof_solve.py 3 12 > gpurun_out/u2_prof_plain.log 2>&1 && \
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 10 -c 1 -o gpurun_out/u2_prof_cfg3 -f python tools/prof_solve.py 3 12 > gpurun_out/u2_ncu_full.log 2>&1
echo ncu=$?
ncu -i gpurun_out/u2_prof_cfg3.ncu-rep --page source --csv --print-source sass > gpurun_out/u2_prof_cfg3_sass.csv 2>/dev/null
ncu -i gpurun_out/u2_prof_cfg3.ncu-rep --page details --csv > gpurun_out/u2_prof_cfg3_details.csv 2>/dev/null
ls -la gpurun_out | head -40
