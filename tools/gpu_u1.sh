#!/bin/bash
# round-2 session 4: cfg4 oracle fixture on the box's host cores (background, oracle/ only)
# while the GPU runs the group-progress-bound A/B (results of gpu_t2.sh were lost)
cd "$(dirname "$0")/.."
free -g | head -2; nproc
( timeout 4500 python tests/golden/make_oracle_fixtures.py cfg4 > gpurun_out/u1_fixture.log 2>&1; echo fixture=$? >> gpurun_out/u1_fixture.log; cp -f tests/golden/oracle_cfg4.npz gpurun_out/ 2>/dev/null ) &
FIX=$!
sleep 20; cat gpurun_out/u1_fixture.log
ROUNDS=2 REPS=2 timeout 1500 python tools/env_ab.py 5 20 base: lag1:HQ_GLAG=1 lag2:HQ_GLAG=2 lag4:HQ_GLAG=4 g10l1:HQ_GROUP_BITS=10,HQ_GLAG=1 g10l2:HQ_GROUP_BITS=10,HQ_GLAG=2 > gpurun_out/u1_ab_cfg5.jsonl 2>&1; echo ab5=$?
cat gpurun_out/u1_ab_cfg5.jsonl
ROUNDS=2 REPS=2 timeout 900 python tools/env_ab.py 4 40 base: lag1:HQ_GLAG=1 lag2:HQ_GLAG=2 g10l1:HQ_GROUP_BITS=10,HQ_GLAG=1 > gpurun_out/u1_ab_cfg4.jsonl 2>&1; echo ab4=$?
cat gpurun_out/u1_ab_cfg4.jsonl
wait $FIX
cat gpurun_out/u1_fixture.log; ls -la gpurun_out/
