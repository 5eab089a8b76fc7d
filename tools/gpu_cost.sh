for m in 0 1 2; do echo "== HQ_COST=$m"; HQ_COST=$m HQ_LIB=variants/libhq_wt.so timeout 300 python tools/warp_timing.py 3 2>&1 | grep "CTA max\|pred max"; done
VARIANTS="s11 s11@HQ_COST=1 s11@HQ_COST=2 s11@HQ_COST=1@HQ_COST_BASE=150 s11@HQ_COST=1@HQ_COST_BASE=400" CFG=3 REPS=4 bash tools/gpu_ab.sh
