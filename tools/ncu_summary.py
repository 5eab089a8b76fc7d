"""Summarise an `ncu --set full` capture of the sweep kernel into profiles/ncu_summary.json
(read by bench.py for roofline.traffic, the binding unit and the FP64 / issue fractions).

  python tools/ncu_summary.py REPORT.ncu-rep CFG [KERNEL_REGEX]

Per config: the mean over the captured k_sweep3 launches of
  dram_bytes_per_launch  dram__bytes_read.sum + dram__bytes_write.sum
  dram_throughput_frac   gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed / 100
  issue_active           smsp__issue_active.avg.pct_of_peak_sustained_active / 100
  fp64_pipe_frac         sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active / 100
  warp_inst_per_launch   smsp__inst_executed.sum
  l2_hit_rate            lts__t_sector_hit_rate.pct / 100
Development aid (run here on a report brought back from the GPU box)."""
import csv
import io
import json
import os
import re
import subprocess
import sys

rep, cfg = sys.argv[1], int(sys.argv[2])
kre = re.compile(sys.argv[3] if len(sys.argv) > 3 else "k_sweep3")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9,
         "second": 1, "cycle": 1, "inst": 1, "%": 1, "": 1, "Kcycle": 1e3, "Mcycle": 1e6, "Kinst": 1e3,
         "Minst": 1e6, "Ginst": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1}


def num(d, k):
    if k not in d or d[k] in ("", "n/a"):
        return None
    v = float(d[k].replace(",", ""))
    return v * SCALE.get(units[hdr.index(k)], 1)


launches = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if not kre.search(d.get("Kernel Name", "")):
        continue
    cyc = num(d, "smsp__cycles_elapsed.avg")
    # FP64 thread instructions per cycle (fused DFMA + non-fused DADD, DMUL) x elapsed cycles
    fp64 = 0.0
    for k in ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
              "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
              "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed"):
        fp64 += (num(d, k) or 0.0) * (cyc or 0.0)
    e = dict(
        kernel=d["Kernel Name"],
        gpu_time_s=num(d, "gpu__time_duration.sum"),
        dram_bytes_per_launch=(num(d, "dram__bytes_read.sum") or 0.0) + (num(d, "dram__bytes_write.sum") or 0.0),
        dram_throughput_frac=(num(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed") or 0.0) / 100,
        issue_active=(num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active") or 0.0) / 100,
        warp_inst_per_launch=num(d, "smsp__inst_executed.sum") or num(d, "sm__inst_executed.sum"),
        l2_hit_rate=(num(d, "lts__t_sector_hit_rate.pct") or 0.0) / 100,
        registers=num(d, "launch__registers_per_thread"),
        warps_active=(num(d, "sm__warps_active.avg.pct_of_peak_sustained_active") or 0.0) / 100,
        fp64_thread_inst=fp64,
        fp64_pipe_frac=(num(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") or 0.0) / 100,
    )
    launches.append(e)
if not launches:
    sys.exit("no launch of " + kre.pattern + " in " + rep)


def mean(k):
    v = [x[k] for x in launches if x[k] is not None]
    return sum(v) / len(v) if v else None


path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_summary.json")
db = json.load(open(path)) if os.path.exists(path) else {}
ent = {k: mean(k) for k in launches[0] if k != "kernel"}
ent["launch_us_under_ncu"] = ent.pop("gpu_time_s") * 1e6 if ent.get("gpu_time_s") else None
ent.update(kernel=launches[0]["kernel"], launches=len(launches), source=os.path.basename(rep))
db[f"cfg{cfg}"] = ent
json.dump(db, open(path, "w"), indent=1, sort_keys=True)
print(json.dumps(ent, indent=1))
