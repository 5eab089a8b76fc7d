#!/bin/bash
# regenerate the committed ncu summaries of the k_sweep3 capture (gpurun_out/prof_cfg3.ncu-rep)
set -e
R=gpurun_out/prof_cfg3.ncu-rep
O=profiles/r01
ncu -i $R --page details --csv > $O/ncu_k_sweep3_cfg3_details.csv 2>/dev/null
ncu -i $R --page source --csv --print-source cuda,sass > /tmp/ncu_src.csv 2>/dev/null
python tools/ncu_line_summary.py /tmp/ncu_src.csv 60 > $O/ncu_k_sweep3_cfg3_lines.txt
ncu -i $R --page source --csv --print-source sass > /tmp/ncu_sass.csv 2>/dev/null
python tools/ncu_sass_summary.py /tmp/ncu_sass.csv > $O/ncu_k_sweep3_cfg3_sass.txt
ncu -i $R --page raw --csv > /tmp/ncu_raw.csv 2>/dev/null
python3 - <<'PY' > $O/ncu_k_sweep3_cfg3_stalls.txt
import csv
rows = list(csv.reader(open('/tmp/ncu_raw.csv')))
h = rows[0]
d = dict(zip(h, rows[2]))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]
for k in keys:
    print(f"{k:60s} {d.get(k, '?')}")
print("stall reasons (pc samples):")
st = []
for k, v in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            st.append((float(v.replace(",", "")), k))
        except ValueError:
            pass
tot = sum(x for x, _ in st)
for v, k in sorted(st, reverse=True)[:14]:
    print(f"  {k[len('smsp__pcsamp_warps_issue_stalled_'):]:28s} {v:8.0f} {100 * v / tot:5.1f}%")
PY
cat $O/ncu_k_sweep3_cfg3_stalls.txt
