CFG=3 VARIANTS="auto2 auto prev" bash tools/gpu_ab.sh
CFG=4 REPS=2 VARIANTS="auto2 prev" bash tools/gpu_ab.sh
