#!/bin/bash
# group progress bound: correctness at N = 23, then same-box A/B at cfg5 / cfg4
cd "$(dirname "$0")/.."
free -g | head -2; nproc
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x --timeout 600 -k "group_lag or tile_orders" > gpurun_out/t2_pytest.log 2>&1; echo pytest=$?
tail -5 gpurun_out/t2_pytest.log
ROUNDS=2 REPS=2 timeout 1500 python tools/env_ab.py 5 20 base: lag1:HQ_GLAG=1 lag2:HQ_GLAG=2 lag4:HQ_GLAG=4 g10l1:HQ_GROUP_BITS=10,HQ_GLAG=1 g10l2:HQ_GROUP_BITS=10,HQ_GLAG=2 g9l2:HQ_GROUP_BITS=9,HQ_GLAG=2 > gpurun_out/t2_ab_cfg5.jsonl 2>&1; echo ab5=$?
cat gpurun_out/t2_ab_cfg5.jsonl
ROUNDS=2 REPS=2 timeout 900 python tools/env_ab.py 4 40 base: lag1:HQ_GLAG=1 lag2:HQ_GLAG=2 g10l1:HQ_GROUP_BITS=10,HQ_GLAG=1 g10l2:HQ_GROUP_BITS=10,HQ_GLAG=2 > gpurun_out/t2_ab_cfg4.jsonl 2>&1; echo ab4=$?
cat gpurun_out/t2_ab_cfg4.jsonl
