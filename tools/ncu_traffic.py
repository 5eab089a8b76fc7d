"""Write profiles/ncu_traffic.json from an `ncu --set full` report of the sweep kernel:
DRAM bytes (read + write) per k_sweep3 launch.  Development aid:
  python tools/ncu_traffic.py REPORT.ncu-rep CFG"""
import csv
import io
import json
import os
import subprocess
import sys

rep, cfg = sys.argv[1], int(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
units = rows[1]
vals = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if "k_sweep3" not in d.get("Kernel Name", ""):
        continue
    def num(k):
        v = float(d[k].replace(",", ""))
        u = units[hdr.index(k)]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3,
                    "nsecond": 1e-9, "second": 1}.get(u, 1)
    vals.append((num("dram__bytes_read.sum") + num("dram__bytes_write.sum"), num("gpu__time_duration.sum"),
                 d["Kernel Name"]))
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
db[f"cfg{cfg}"] = dict(dram_bytes_per_launch=sum(v[0] for v in vals) / len(vals),
                       launch_seconds_under_ncu=sum(v[1] for v in vals) / len(vals), launches=len(vals),
                       kernel=vals[0][2], source=os.path.basename(rep))
json.dump(db, open(path, "w"), indent=1)
print(db[f"cfg{cfg}"])
