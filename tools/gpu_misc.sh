M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
for v in s12 s12pol; do echo "== $v"; HQ_LIB=variants/libhq_$v.so timeout 300 ncu --metrics $M --clock-control none -k regex:k_sweep3 -s 40 -c 1 python tools/prof_solve.py 3 30 2>&1 | grep -E "dram__|gpu__time|lts__"; done
VARIANTS="s12 s12pol" CFG=3 REPS=4 bash tools/gpu_ab.sh
