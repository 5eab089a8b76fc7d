"""Summarise an ncu --page source --print-source sass CSV: instructions and
stall samples per opcode and the hottest instructions.  Development aid."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
ix = {k: i for i, k in enumerate(hdr)}
ops = collections.Counter()
stall = collections.Counter()
tot_inst = 0
tot_samp = 0
hot = []
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        break
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ops[op] += n
    stall[op] += s
    tot_inst += n
    tot_samp += s
    hot.append((s, n, r[0], src))
print(f"total warp instructions {tot_inst}, stall samples {tot_samp}")
print("opcode               inst%   stall%")
for op, n in ops.most_common(30):
    print(f"{op:18s} {100*n/tot_inst:7.2f} {100*stall[op]/max(tot_samp,1):7.2f}")
print("hottest by samples:")
for s, n, a, src in sorted(hot, reverse=True)[:40]:
    print(f"{s:7d} {n:10d} {a[-5:]} {src}")
