#!/bin/bash
# register / spill report of the k_sweep3 instantiations (development helper)
#   tools/ptxas_v3.sh [extra nvcc flags]
cd "$(dirname "$0")/../paper_2603_03019_b200/csrc" && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xptxas -v "$@" -c hq_v3.cu -o /tmp/hq_v3.o 2>&1 | python3 -c '
import re, sys
name = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function .(_Z\w+)", line)
    if m:
        k = re.search(r"k_sweep3ILi(\d)ELb(\d)ELb(\d)E(?:Lb(\d))?", m.group(1))
        name = f"k_sweep3<{k.group(1)},{k.group(2)},{k.group(3)},{k.group(4)}>" if k else m.group(1)[:40]
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name: sp = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        print(f"{name:40s} regs {m.group(1):>4s}  spill st/ld {sp[0]}/{sp[1]}")
        name = None
    if "error" in line: print(line.rstrip())
'
