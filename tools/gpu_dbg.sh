CFG=3 REPS=3 VARIANTS="hdr2 hdr2@cta hdr2@warp" bash tools/gpu_ab.sh
CFG=4 REPS=2 VARIANTS="hdr2 hdr2@cta hdr2@warp" bash tools/gpu_ab.sh
