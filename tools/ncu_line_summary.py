"""Per-CUDA-source-line instruction counts and stall samples from
`ncu -i X --page source --csv --print-source cuda,sass`.  Development aid."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
res = []
hdr = None
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0].isdigit():
        continue
    if r[2] != "-":   # sass rows carry an address; cuda-line rows have '-'
        continue
    try:
        samples = int(r[4] or 0)
        inst = int(r[7] or 0)
    except ValueError:
        continue
    res.append((inst, samples, int(r[0]), r[1][:110]))
ti = sum(x[0] for x in res)
ts = sum(x[1] for x in res)
print(f"total warp instr {ti}  samples {ts}")
for inst, s, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{100*inst/ti:6.2f}% {100*s/max(ts,1):6.2f}%  L{ln:4d} {src}")
