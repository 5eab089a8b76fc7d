#!/bin/bash
# DRAM traffic of the device-resident solve at cfg5 (natural order, dynamic units) vs host loop
cd "$(dirname "$0")/.."
timeout 300 python tools/prof_dev.py 5 1 > gpurun_out/s4_plain.log 2>&1 && \
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_solve3 -c 1 --csv --log-file gpurun_out/s4_ncu_solve5.csv python tools/prof_dev.py 5 1 > gpurun_out/s4_ncu.log 2>&1
for u in 1 4 16; do for hn in 14; do
HQ_UNIT=$u HQ_DEBUG_CTL=1 timeout 300 python tools/prof_dev.py 5 3 >> gpurun_out/s4_units.log 2>&1
done; done
echo done
